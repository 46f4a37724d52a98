export TC_TIMEOUT_MS=20000
mkdir -p gpurun_out/r01
timeout 900 python -m pytest tests/test_gpu_bucketed.py -x -q 2>&1 | tail -2
for NP in 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 29551 bench_overlap.py --ratio 1.0 > gpurun_out/r01/overlap_p$NP.log 2>&1; echo "rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 29552 bench_overlap.py --ratio 3.0 --bucket-mb 10 >> gpurun_out/r01/overlap_p$NP.log 2>&1; echo "rc=$?"
grep bench gpurun_out/r01/overlap_p$NP.log
done
