summ() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['achieved'], d['solve_roofline']['frac'], d['e2e']['value'], d.get('timestep',{}).get('ms_per_step'))"; }
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1 >> gpurun_out/ab.txt
for c in 2 5 3; do
for v in "HPS_KSPLIT_CLUSTER=0" "HPS_KSPLIT_CLUSTER=1"; do
  echo "== cfg$c $v" >> gpurun_out/ab.txt
  env $v timeout 300 python bench.py --config $c --skip-cpu 2>&1 | summ >> gpurun_out/ab.txt 2>&1
done; done
python tools/sweep_steps.py --config 2 > gpurun_out/steps_cfg2.txt 2>&1
cat gpurun_out/ab.txt
