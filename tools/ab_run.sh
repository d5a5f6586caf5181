timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -1 >> gpurun_out/ab.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:leaf_assemble --log-file gpurun_out/asm.csv python tools/ncu_target.py --config 3 --solves 0 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:leaf_assemble --log-file gpurun_out/asm5.csv python tools/ncu_target.py --config 5 --solves 0 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/asm.csv 1 >> gpurun_out/ab.txt; python tools/launch_summary.py gpurun_out/asm5.csv 1 >> gpurun_out/ab.txt
for c in 3 5; do timeout 300 python tools/profile_build.py --config $c 2>&1 | grep -E "leaf-build" >> gpurun_out/ab.txt; done
cat gpurun_out/ab.txt
