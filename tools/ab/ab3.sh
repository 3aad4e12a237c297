python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_golden.py tests/test_gpu_rect.py tests/test_gpu_fullsize_ops.py tests/test_gpu_configs.py -x -q 2>&1 | tail -3
HTG_FDM_SYM=1 python -m pytest tests/test_gpu_fullsize_ops.py -x -q 2>&1 | tail -2
python tools/fdm_ab.py
HTG_FDM_TEAM=2 python tools/fdm_ab.py
HTG_FDM_SYM=1 python tools/fdm_ab.py
