timeout 300 python tools/profile_build.py --config 5 2>&1 | grep -E "merge d[0-4] " >> gpurun_out/ab.txt
timeout 300 python tools/profile_build.py --config 3 2>&1 | grep -E "merge d[0-4] |leaf-build" >> gpurun_out/ab.txt
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1 >> gpurun_out/ab.txt
cat gpurun_out/ab.txt
