set -x
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo ref rc=$?
HTG_ND_TIMES=1 HTG_SETUP_TIMES=1 python tools/run_once.py --what step --reps 1 > gpurun_out/final_setup.log 2>&1
bash tools/profile_round.sh > gpurun_out/final_profile.log 2>&1; echo prof rc=$?
