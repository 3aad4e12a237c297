for v in k1_u4 k1_c58 k1_c56 k1_c62; do
AB_WL=160 HTG_LIB=exp/$v.so python tools/fdm_ab.py 2>&1 | tail -1
done
AB_WL=160 python tools/fdm_ab.py
