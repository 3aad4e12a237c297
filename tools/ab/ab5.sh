for e in 1 2 3; do echo "== exp $e"
HTG_LIB=exp/fexp$e.so python tools/run_once.py --what sweep --reps 3 --wavelengths 160 2>&1 | grep "fdm trace" | tail -32 | grep "part 0" | grep "cta 70" | sort -k4n -k6n | tail -8
done
