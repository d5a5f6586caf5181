for v in "HPS_GJ_NARROW128=0" "HPS_GJ_NARROW128=1"; do
echo "== $v" >> gpurun_out/ab.txt
env $v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:gemm_big --log-file gpurun_out/g.csv python tools/ncu_target.py --config 3 --solves 0 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/g.csv 1 | grep "1024)" | head -4 >> gpurun_out/ab.txt
env $v timeout 300 python tools/profile_build.py --config 3 2>&1 | grep -E "leaf-build" >> gpurun_out/ab.txt
done
HPS_GJ_NARROW128=1 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> gpurun_out/ab.txt
cat gpurun_out/ab.txt
