# Round-1 evidence run: bench at N=1 and N=2, ncu launch list and one full capture of the top kernel.
export TC_TIMEOUT_MS=10000
mkdir -p gpurun_out/r01
timeout 600 python bench.py > gpurun_out/r01/bench_n1.log 2>&1; echo "bench n1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 > gpurun_out/r01/bench_n2.log 2>&1; echo "bench n2 rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/r01/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01/launches_n1.csv $CMD > gpurun_out/r01/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_local -s 3 -c 1 -o gpurun_out/r01/prof_local $CMD > gpurun_out/r01/ncu_full.log 2>&1; echo "ncu full rc=$?"
