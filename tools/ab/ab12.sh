python tools/fdm_ab.py
HTG_LIB=exp/x_tgw1.so python tools/fdm_ab.py
HTG_LIB=exp/x_tgw3.so python tools/fdm_ab.py
HTG_FDM_TEAM=2 AB_WL=80 python tools/fdm_ab.py
HTG_FDM_TEAM=4 AB_WL=80 python tools/fdm_ab.py
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_ops.py tests/test_gpu_rect.py tests/test_gpu_ref_golden.py -x -q 2>&1 | tail -2
