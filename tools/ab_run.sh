summ() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['solve_roofline']['frac'])"; }
for c in 2 5 3; do
for v in "HPS_SPLIT_CTAS=600" "HPS_SPLIT_CTAS=300" "HPS_SPLIT_CTAS=1200" "HPS_SPLIT_BYTES=2e6" "HPS_SPLIT_BYTES=8e6"; do
  echo "== cfg$c $v" >> gpurun_out/ab.txt
  env $v timeout 300 python bench.py --config $c --skip-cpu --steps 200 2>&1 | summ >> gpurun_out/ab.txt 2>&1
done; done
cat gpurun_out/ab.txt
