for i in 1 2; do timeout 300 python tools/profile_build.py --config 5 2>&1 | grep -E "build .* s \(rep|leaf-build" >> gpurun_out/ab.txt; done
cat gpurun_out/ab.txt
