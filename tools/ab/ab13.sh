python tools/fdm_ab.py
HTG_FDM_TEAM=3 HTG_FDM_NTEAMS=6 AB_WL=80 python tools/fdm_ab.py
HTG_FDM_TEAM=2 AB_WL=80 python tools/fdm_ab.py
HTG_FDM_TEAM=4 AB_WL=80 python tools/fdm_ab.py
HTG_FDM_TEAM=2 HTG_FDM_NTEAMS=6 AB_WL=80 python tools/fdm_ab.py
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_ops.py -x -q 2>&1 | tail -2
