summ() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['solve_roofline']['frac'], d.get('timestep',{}).get('ms_per_step'))"; }
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 >> gpurun_out/ab.txt
for v in "HPS_DMMA_MULTI=0" "HPS_DMMA_MULTI=1"; do
  echo "== cfg5 16rhs $v" >> gpurun_out/ab.txt
  env $v timeout 300 python bench.py --config 5 --nrhs 16 --skip-cpu --steps 100 2>&1 | summ >> gpurun_out/ab.txt 2>&1
done
python tools/sweep_steps.py --config 5 --nrhs 16 > gpurun_out/steps_cfg5_16.txt 2>&1
cat gpurun_out/ab.txt
