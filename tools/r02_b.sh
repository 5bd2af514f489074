mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/b_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_f3.py tests/test_gpu_f4.py tests/test_bench_contract.py -x -q -m gpu > gpurun_out/b_tests.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-f3 --no-f4 --no-latency > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err
bash tools/sanitize.sh
