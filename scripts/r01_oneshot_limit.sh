# one-shot vs TMA two-shot at 1 and 4 MiB, every tensor count, p = 4 and 3 (current build)
mkdir -p gpurun_out
TR="timeout 300 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29515"
for N in 4 3; do
  $TR --nproc-per-node $N bench_sweep.py --sizes 5,6,7 > gpurun_out/os_auto_p$N.jsonl 2>/dev/null; echo auto$N $?
  $TR --nproc-per-node $N bench_sweep.py --sizes 5,6,7 --algo 6 --oneshot 0 --ll 0 > gpurun_out/os_tma_p$N.jsonl 2>/dev/null; echo tma$N $?
done
