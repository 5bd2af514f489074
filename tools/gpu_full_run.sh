mkdir -p gpurun_out
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-exact --no-f1 --no-f3 --no-f4 --no-c2 --no-c5 --no-latency"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_l.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"window_kernel|frame_kernel" -s 6 -c 2 -o gpurun_out/prof_r01 -f $CMD > gpurun_out/ncu_f.log 2>&1
nproc; lscpu | grep "Model name"
