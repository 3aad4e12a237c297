HTG_FDM_TEAM=3 HTG_FDM_NTEAMS=8 python tools/fdm_ab.py
HTG_FDM_TEAM=3 HTG_FDM_NTEAMS=7 python tools/fdm_ab.py
python tools/fdm_ab.py
HTG_FDM_TEAM=3 HTG_FDM_NTEAMS=8 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_ops.py -x -q 2>&1 | tail -2
