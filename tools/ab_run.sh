for c in 5 2 3; do python tools/build_host_profile.py $c 2>&1 | grep "^build" >> gpurun_out/ab.txt; done
python tools/build_host_profile.py 5 2>&1 | grep -v "^$" | sed -n 3,20p >> gpurun_out/ab.txt
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 >> gpurun_out/ab.txt
cat gpurun_out/ab.txt
