python tools/fdm_ab.py
for v in v_s0c0d28 v_s0c0d4 v_s0c1d28 v_s0c1d4 v_s1c0d28 v_s1c0d4 v_s1c1d28 v_s1c1d4; do
HTG_LIB=exp/$v.so python tools/fdm_ab.py
done
HTG_SETUP_TIMES=1 python tools/run_once.py --what step --reps 1 2>&1 | grep "htg setup"
