python -m pytest tests/test_gpu_fdm_shapes.py tests/test_gpu_parity.py tests/test_gpu_fullsize_ops.py tests/test_gpu_rect.py -x -q 2>&1 | tail -2
python tools/fdm_ab.py
HTG_LIB=exp/nomerge.so python tools/fdm_ab.py
HTG_FDM_TEAM=2 AB_WL=80 python tools/fdm_ab.py
HTG_FDM_TEAM=4 AB_WL=80 python tools/fdm_ab.py
HTG_FDM_TEAM=3 HTG_FDM_NTEAMS=6 AB_WL=80 python tools/fdm_ab.py
AB_WL=40,120 python tools/fdm_ab.py
AB_WL=40,120 HTG_LIB=exp/nomerge.so python tools/fdm_ab.py
