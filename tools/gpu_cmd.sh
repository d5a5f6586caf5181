O=gpurun_out
for nc in 16 8; do for mr in 128 32; do
echo "NC=$nc MINR=$mr" >> $O/ab5.log
HPS_TMA_NC=$nc HPS_TMA_MINR=$mr timeout 300 python tools/sweep_steps.py --config 5 --nrhs 16 > $O/steps5_nc${nc}_mr${mr}.log 2>&1
grep -E "items= 16384|sum" $O/steps5_nc${nc}_mr${mr}.log >> $O/ab5.log
done; done
timeout 600 python -m pytest tests/test_gpu_cfg5_trajectory.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > $O/t4.log 2>&1
