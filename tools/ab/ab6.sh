python -m pytest tests/test_gpu_parity.py tests/test_gpu_rect.py tests/test_gpu_fullsize_ops.py tests/test_gpu_ref_golden.py -x -q 2>&1 | tail -2
python tools/fdm_ab.py
HTG_LIB=exp/noconst.so python tools/fdm_ab.py
HTG_LIB=exp/nosym.so python tools/fdm_ab.py
HTG_FDM_TEAM=2 python tools/fdm_ab.py
HTG_FDM_TEAM=3 HTG_FDM_NTEAMS=5 python tools/fdm_ab.py
