# A/B of the FDM kernel variants at cfg4 (bench.py without the CPU/dense/cfg3 legs)
# usage: bash tools/ab_fdm.sh "name1:ENV=.. ENV=.." "name2:..."
python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_golden.py -x -q > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
HTG_FDM_GROUPK=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ref_golden.py -x -q > gpurun_out/t4.log 2>&1; echo rc=$? >> gpurun_out/t4.log
for spec in "$@"; do
  name=${spec%%:*}; envs=${spec#*:}
  env $envs python bench.py --no-cpu-baseline --no-dense --no-cfg3 --steps 30 > "gpurun_out/ab_$name.log" 2>&1
done
