HTG_ND_TIMES=1 HTG_SETUP_TIMES=1 python tools/run_once.py --what step --reps 1 2>&1 | grep -E "htg|ok"
python bench.py --no-cpu-baseline --no-dense > gpurun_out/share_bench.json 2> gpurun_out/share_bench.err; echo rc=$?
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
