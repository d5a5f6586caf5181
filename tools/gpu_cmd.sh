O=gpurun_out
timeout 120 tools/tma_stream > $O/tma.log 2>&1
timeout 300 python tools/e2e_parts.py 2 > $O/e2e.log 2>&1
timeout 300 python -m pytest tests/test_gpu_api.py -q -p no:cacheprovider > $O/t2.log 2>&1
timeout 300 python tools/profile_build.py --config 2 > $O/pb2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gj_fused -c 1 -o $O/gjf2 python tools/ncu_target.py --config 2 --solves 0 > $O/ncu_gjf2.log 2>&1
timeout 120 ncu -i $O/gjf2.ncu-rep --page details --csv > $O/gjf2_details.csv 2>&1
timeout 120 python tools/ncu_hot.py $O/gjf2.ncu-rep 40 > $O/gjf2_hot.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-extras > $O/b2.log 2>&1
rm -f $O/*.ncu-rep
