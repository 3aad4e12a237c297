python tools/fdm_ab.py
for v in w_tgw2 w_du8 w_swapb w_m4 w_tgw2swapb w_ksplit2 w_swapbdu8; do
AB_WL=160 HTG_LIB=exp/$v.so python tools/fdm_ab.py
done
HTG_SETUP_TIMES=1 python tools/run_once.py --what step --reps 1 2>&1 | grep "htg setup"
