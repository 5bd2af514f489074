mkdir -p gpurun_out
IEDS_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --windows 2000 --c5-windows 2000 --no-exact --no-c2 > gpurun_out/n2.json 2> gpurun_out/n2.err
echo "rc=$?" >> gpurun_out/n2.err
