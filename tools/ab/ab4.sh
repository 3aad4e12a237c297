python -m pytest tests/test_gpu_parity.py tests/test_gpu_rect.py -x -q 2>&1 | tail -2
python tools/fdm_ab.py
HTG_LIB=exp/comb2.so python tools/fdm_ab.py
HTG_LIB=exp/comb8.so python tools/fdm_ab.py
for wl in 80 160; do
HTG_LIB=exp/fdmtrace.so python tools/run_once.py --what sweep --reps 3 --wavelengths $wl 2>&1 | grep "fdm trace" | tail -32 | grep "part 0" | sort -k4n -k6n | tail -8
done
