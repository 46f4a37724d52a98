# Evidence after the p=1 TMA stream: bench N=1, ncu launch list, one full capture of k_local_tma.
export TC_TIMEOUT_MS=10000
mkdir -p gpurun_out/r01d
timeout 600 python bench.py > gpurun_out/r01d/bench_n1.log 2>&1; echo "bench n1 rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/r01d/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01d/launches_n1.csv $CMD > gpurun_out/r01d/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_local_tma -s 3 -c 1 -o gpurun_out/r01d/prof_local_tma $CMD > gpurun_out/r01d/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/r01d/prof_local_tma.ncu-rep --page raw --csv > gpurun_out/r01d/ncu_full_raw.csv 2>/dev/null; echo "export rc=$?"
