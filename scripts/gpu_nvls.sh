export TC_TIMEOUT_MS=10000
NP=${NP:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 29514"
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -s 2>&1 | grep -E "passed|failed|Error|error|symmetric|assert" | head -20
for algo in 1 4; do
  TC_DEBUG=1 timeout 300 $TR tools/phase_probe.py --sym --algo $algo 2>&1 | grep -E "rank|libtc" | head -8
done
for algo in 0 4; do
timeout 600 $TR bench.py --gpus $NP --no-e2e --algo $algo > gpurun_out/bench_n${NP}_sym_a$algo.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_n${NP}_sym_a$algo.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ['t_us','busbw_gbs','allreduce_only','nccl_allreduce_flat','easgd']}, d['config']['algo'])"
done
