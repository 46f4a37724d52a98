export TC_TIMEOUT_MS=20000
NP=4
mkdir -p gpurun_out/r01
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 29561"
timeout 300 $TR tools/phase_probe.py --sym --algo 1 2>&1 | grep -E "rank" | head -8
timeout 900 $TR bench_sweep.py --sizes 6,7,8,9,10 --tensors 1,161 --out gpurun_out/r01/sweep_p4_mid.jsonl > /dev/null 2>&1; echo "sweep rc=$?"
timeout 600 $TR bench.py --gpus $NP --no-e2e > gpurun_out/r01/bench_n4b.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r01/bench_n4b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ['t_us','busbw_gbs','allreduce_only','nccl_allreduce_flat','easgd']}, d['config']['algo'])"
