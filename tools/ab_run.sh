summ() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['solve_roofline']['frac'])"; }
for v in "HPS_PDL=1" "HPS_PDL=0"; do
  echo "== cfg2 $v" >> gpurun_out/ab.txt
  env $v timeout 300 python bench.py --config 2 --skip-cpu --steps 200 2>&1 | summ >> gpurun_out/ab.txt 2>&1
done
cat gpurun_out/ab.txt
