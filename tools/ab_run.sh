timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> gpurun_out/ab.txt
for c in 5 3; do timeout 300 python tools/profile_build.py --config $c 2>&1 | grep -E "merge d[0-4] |leaf-build" >> gpurun_out/ab.txt; done
python tools/build_reps.py 2>&1 | tail -7 >> gpurun_out/ab.txt
cat gpurun_out/ab.txt
