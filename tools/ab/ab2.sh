./tools/dmma_roles
HTG_LIB=exp/swapb.so python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
python tools/fdm_ab.py
HTG_LIB=exp/swapb.so python tools/fdm_ab.py
HTG_LIB=exp/swapb.so HTG_FDM_TEAM=3 HTG_FDM_NTEAMS=5 python tools/fdm_ab.py
HTG_LIB=exp/swapbtrace.so python tools/run_once.py --what sweep --reps 3 --wavelengths 160 2>&1 | grep "fdm trace" | tail -32 | grep "part 0" | sort -k4n -k6n
