python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py > gpurun_out/last_bench.json 2> gpurun_out/last_bench.err; echo bench rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/last_ref.json 2> gpurun_out/last_ref.err; echo ref rc=$?
python -c "import __graft_entry__ as g; g.smoke()"
