timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1 >> gpurun_out/ab.txt
for c in 3 5 2; do timeout 300 python tools/profile_build.py --config $c 2>&1 | grep -E "leaf-build" >> gpurun_out/ab.txt; done
python tools/build_reps.py 2>&1 | grep -E "^(5|2) 4" >> gpurun_out/ab.txt
cat gpurun_out/ab.txt
