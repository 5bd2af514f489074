# Round evidence on one B200 (profiles/README.md): the GPU test suite, the default bench line, the
# reference arm, an ncu launch list of the timed hot path and one ncu --set full capture of the
# frame and window kernels.  Everything lands in gpurun_out/.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/full_tests.log 2>&1
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-exact --no-f1 --no-f3 --no-f4 --no-c2 --no-c5 --no-c4-r1 --no-latency"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_l.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"window_kernel|frame_kernel" -s 6 -c 2 -o gpurun_out/prof_full -f $CMD > gpurun_out/ncu_f.log 2>&1
nproc > gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt
