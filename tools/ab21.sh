timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ab21_tests.txt 2>&1
timeout 600 python bench.py --skip-cpu > gpurun_out/ab21_bench.txt 2>&1
