mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest.log 2>&1
timeout 600 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
which compute-sanitizer >> gpurun_out/r02_smi.txt 2>&1; ls /usr/local/cuda/bin | grep -i sanit >> gpurun_out/r02_smi.txt
