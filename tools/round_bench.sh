# Bench lines only (see round_profiles.sh for the full pass)
R=${R:-r04}
O=gpurun_out
for c in 1 2 3 4 5; do timeout 600 python bench.py --config $c > $O/${R}_bench_cfg$c.log 2>&1; tail -1 $O/${R}_bench_cfg$c.log > $O/${R}_bench_cfg$c.json; done
timeout 600 python bench.py --config 5 --nrhs 16 --skip-cpu > $O/${R}_bench_cfg5_16rhs.log 2>&1; tail -1 $O/${R}_bench_cfg5_16rhs.log > $O/${R}_bench_cfg5_16rhs.json
timeout 900 python -m pytest tests -m gpu -q > $O/${R}_pytest_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/${R}_smoke.txt 2>&1
