O=gpurun_out
timeout 300 python tools/debug_fold.py 8 4 > $O/dbg_fold.log 2>&1
timeout 300 python tools/debug_fold.py 16 16 >> $O/dbg_fold.log 2>&1
timeout 900 python -m pytest tests/test_gpu_cfg5_trajectory.py tests/test_timestepping.py -q -p no:cacheprovider -x > $O/t11.log 2>&1
timeout 600 python bench.py --config 5 --steps 20 --skip-cpu > $O/b5.log 2>&1
