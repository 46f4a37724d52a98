# tests, p=NP phase timings, bench at N=NP and N=1, ncu launch list + full capture of k_local
export TC_TIMEOUT_MS=10000
NP=${NP:-4}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 29517"
mkdir -p gpurun_out/r01b
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for algo in 1 3; do
  timeout 300 $TR tools/phase_probe.py --sym --algo $algo 2>&1 | grep -E "rank" | head -8
done
timeout 600 $TR bench.py --gpus $NP > gpurun_out/r01b/bench_n$NP.log 2>&1; echo "bench n$NP rc=$?"
timeout 600 python bench.py > gpurun_out/r01b/bench_n1.log 2>&1; echo "bench n1 rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/r01b/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01b/launches_n1.csv $CMD > gpurun_out/r01b/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_local -s 3 -c 1 -o gpurun_out/r01b/prof_local $CMD > gpurun_out/r01b/ncu_full.log 2>&1; echo "ncu full rc=$?"
