# Round-1 evidence (final kernels): smoke, tests, bench N=1 and N=2, ncu launch list + full capture of the p=1 kernel
export TC_TIMEOUT_MS=10000
mkdir -p gpurun_out/r01c
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/r01c/bench_n1.log 2>&1; echo "bench n1 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 > gpurun_out/r01c/bench_n2.log 2>&1; echo "bench n2 rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r01c/bench_ref_n1.log 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/r01c/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01c/launches_n1.csv $CMD > gpurun_out/r01c/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_local -s 3 -c 1 -o gpurun_out/r01c/prof_local $CMD > gpurun_out/r01c/ncu_full.log 2>&1; echo "ncu full rc=$?"
