timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ab25_tests.txt 2>&1
timeout 600 python bench.py --skip-cpu > gpurun_out/ab25_bench.txt 2>&1
timeout 600 python bench.py --config 3 --nrhs 16 --skip-cpu --no-extras > gpurun_out/ab25_bench3.txt 2>&1
