python tools/fdm_ab.py
HTG_SETUP_TIMES=1 python tools/run_once.py --what step --reps 1 2>&1 | grep "htg setup"
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
