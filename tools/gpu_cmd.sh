O=gpurun_out
HPS_STREAM_LEAF=1 timeout 300 python tools/sweep_steps.py --config 5 --nrhs 16 > $O/steps5_streamleaf2.log 2>&1
timeout 300 python tools/sweep_steps.py --config 5 --nrhs 16 > $O/steps5_def2.log 2>&1
HPS_STREAM_LEAF=1 timeout 900 python -m pytest tests/test_gpu_cfg5_trajectory.py -q -p no:cacheprovider -x > $O/t7.log 2>&1
