timeout 300 python tools/sweep_steps.py --config 5 --nrhs 16 > gpurun_out/ab20.txt 2>&1
timeout 300 python tools/sweep_steps.py --config 5 --nrhs 6 2>&1 | tail -1 >> gpurun_out/ab20.txt
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cfg5_trajectory.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ab20_tests.txt 2>&1
