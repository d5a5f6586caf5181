# Measurement pass on the GPU box: tests, bench lines, ncu launch list + full captures.
# Output: gpurun_out/${R}_*  (copied into profiles/ afterwards)
R=${R:-round2a}
O=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $O/${R}_smoke.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/${R}_pytest_gpu.txt 2>&1
timeout 900 python bench.py > $O/${R}_bench_cfg2_default.log 2>&1; tail -1 $O/${R}_bench_cfg2_default.log > $O/${R}_bench_cfg2_default.json
for c in 1 3 4 5; do timeout 600 python bench.py --config $c --no-extras > $O/${R}_bench_cfg$c.log 2>&1; tail -1 $O/${R}_bench_cfg$c.log > $O/${R}_bench_cfg$c.json; done
timeout 600 python bench.py --config 5 --nrhs 16 --skip-cpu --no-extras > $O/${R}_bench_cfg5_16rhs.log 2>&1; tail -1 $O/${R}_bench_cfg5_16rhs.log > $O/${R}_bench_cfg5_16rhs.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/${R}_bench_reference_cfg2.log 2>&1; tail -1 $O/${R}_bench_reference_cfg2.log > $O/${R}_bench_reference_cfg2.json
# launch list of the bench command (cold, serialised: share of the step, not absolute time)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/${R}_bench_cfg2_launches.csv python bench.py --steps 2 --warmup 3 --skip-cpu --no-extras > $O/${R}_ncu_bench.log 2>&1
python tools/launch_summary.py $O/${R}_bench_cfg2_launches.csv 1 > $O/${R}_bench_cfg2_launches_summary.txt 2>&1
# full capture of the dominant solve kernel (leaf downward step, config 2)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o $O/${R}_leafdown_cfg2 python tools/one_step.py --config 2 --reps 1 > $O/${R}_ncu_leafdown.log 2>&1
ncu -i $O/${R}_leafdown_cfg2.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > $O/${R}_leafdown_cfg2_raw.csv 2>&1
python tools/ncu_hot.py $O/${R}_leafdown_cfg2.ncu-rep 30 > $O/${R}_leafdown_cfg2_ncu_source.txt 2>&1
# build: launch lists and phase profiles
for c in 2 3 5; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${R}_build_cfg${c}_launches.csv python tools/ncu_target.py --config $c --solves 0 > /dev/null 2>&1
python tools/launch_summary.py $O/${R}_build_cfg${c}_launches.csv 1 > $O/${R}_build_cfg${c}_launches_summary.txt 2>&1
timeout 300 python tools/profile_build.py --config $c > $O/${R}_profile_build_cfg$c.txt 2>&1
done
timeout 300 python tools/sweep_steps.py --config 2 > $O/${R}_sweep_steps_cfg2.txt 2>&1
timeout 300 python tools/sweep_steps.py --config 5 --nrhs 16 > $O/${R}_sweep_steps_cfg5_16rhs.txt 2>&1
timeout 300 python tools/sweep_steps.py --config 4 > $O/${R}_sweep_steps_cfg4.txt 2>&1
rm -f $O/*.ncu-rep.tmp $O/*.ncu-rep
ls -la $O | tail -40
