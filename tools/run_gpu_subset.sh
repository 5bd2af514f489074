mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_bounds.py tests/test_gpu_variants.py tests/test_gpu_stream.py -q -m gpu > gpurun_out/i_tests.log 2>&1
