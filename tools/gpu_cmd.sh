O=gpurun_out
timeout 300 python tools/sweep_steps.py --config 5 --nrhs 16 > $O/steps5_stream2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_stream -c 1 -o $O/stream_up python tools/ncu_target.py --config 5 --nrhs 16 --solves 1 > $O/ncu_stream.log 2>&1
timeout 120 ncu -i $O/stream_up.ncu-rep --page details --csv > $O/stream_up_details.csv 2>&1
timeout 120 python tools/ncu_hot.py $O/stream_up.ncu-rep 40 > $O/stream_up_hot.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv_tma -c 1 -o $O/tma16b python tools/ncu_target.py --config 5 --nrhs 16 --solves 1 > $O/ncu_tma16b.log 2>&1
timeout 120 ncu -i $O/tma16b.ncu-rep --page raw --csv > $O/tma16b_raw.csv 2>&1
timeout 120 python tools/ncu_hot.py $O/tma16b.ncu-rep 40 > $O/tma16b_hot.txt 2>&1
rm -f $O/*.ncu-rep
