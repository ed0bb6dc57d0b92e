mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gpurun_out/fp64_peak tools/fp64_peak.cu && gpurun_out/fp64_peak > gpurun_out/fp64_peak.json
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/gpu_tests.log 2>&1
echo tests_rc=$?
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_C5.log 2>&1
echo bench_rc=$?
