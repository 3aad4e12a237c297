for v in dotbal w2 w3 w_tgw2swapb; do
HTG_LIB=exp/$v.so python tools/fdm_ab.py
done
HTG_LIB=exp/w2.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_ops.py -x -q 2>&1 | tail -2
