export TC_TIMEOUT_MS=10000
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_n1.log 2>&1; echo "n1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/bench_n2.log 2>&1; echo "n2 rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_local -s 2 -c 1 -o gpurun_out/prof_local $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
tail -3 gpurun_out/bench_n1.log gpurun_out/bench_n2.log
