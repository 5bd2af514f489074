# GPU subset used while iterating: parity + variants + bounds, then a short bench (args: bench flags)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_bounds.py -q -m gpu -x > gpurun_out/sub_tests.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-exact --no-f3 --no-f4 --no-latency "$@" > gpurun_out/sub_bench.json 2> gpurun_out/sub_bench.err
