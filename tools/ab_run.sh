# A/B tuning runs on the GPU box: bench lines under environment knobs
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['achieved'], d['solve_roofline']['frac'])"; }
HPS_FLOW=full timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 >> gpurun_out/ab.txt
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 >> gpurun_out/ab.txt
for c in 2 5; do
for v in "HPS_FLOW=off" "HPS_FLOW=full" "HPS_FLOW=mid" "HPS_FLOW=full HPS_FLOW_CTAS_PER_SM=2" "HPS_FLOW=full HPS_FLOW_UNIT_KB=128"; do
  echo "== cfg$c $v" >> gpurun_out/ab.txt
  env $v timeout 300 python bench.py --config $c --skip-cpu 2>&1 | summ >> gpurun_out/ab.txt 2>&1
done; done
python tools/sweep_steps.py --config 2 > gpurun_out/steps_cfg2.txt 2>&1
cat gpurun_out/ab.txt
