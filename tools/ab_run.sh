timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 >> gpurun_out/ab.txt
for c in 3 5; do timeout 300 python tools/profile_build.py --config $c 2>&1 | grep -E "leaf-build|build .* s \(rep 2\)|merge d[0-4] " >> gpurun_out/ab.txt; done
cat gpurun_out/ab.txt
