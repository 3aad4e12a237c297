python -m pytest tests/test_gpu_parity.py tests/test_gpu_rect.py -x -q 2>&1 | tail -2
HTG_SETUP_TIMES=1 python tools/fdm_ab.py 2>&1 | grep -v "^htg setup:   "
HTG_LIB=exp/nosym.so python tools/fdm_ab.py
HTG_LIB=exp/nosym_du4.so python tools/fdm_ab.py
HTG_LIB=exp/nosym_du8.so python tools/fdm_ab.py
HTG_SETUP_TIMES=1 python tools/run_once.py --what step --reps 1 2>&1 | grep "htg setup"
