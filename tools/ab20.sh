for lib in paper_1612_02736_b200/_hps_b200.so abtest/dmma5/_hps_b200.so abtest/dmma7/_hps_b200.so; do
echo "== $lib"
HPS_B200_LIB=$lib timeout 300 python tools/sweep_steps.py --config 5 --nrhs 16 2>&1 | grep -E "up   items= (16384| 8192|  4096|    64|    32)|down items= *(80|160|320|1024) |sum"
HPS_B200_LIB=$lib timeout 300 python tools/sweep_steps.py --config 3 --nrhs 16 2>&1 | grep -E "sum"
done > gpurun_out/ab20.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cfg5_trajectory.py tests/test_timestepping.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ab20_tests.txt 2>&1
