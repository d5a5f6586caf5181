O=gpurun_out
timeout 300 python tools/debug_gjpair.py > $O/dbg_gjpair.log 2>&1
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "gj" >> $O/t14.log 2>&1; done
