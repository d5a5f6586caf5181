timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 >> gpurun_out/ab.txt
python tools/e2e_parts.py 2 2>&1 | head -3 >> gpurun_out/ab.txt
for c in 2 3 5; do timeout 300 python bench.py --config $c --skip-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['ms_per_step'], d['e2e'])" >> gpurun_out/ab.txt; done
cat gpurun_out/ab.txt
