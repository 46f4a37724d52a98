export TC_TIMEOUT_MS=10000
NP=${NP:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 29512"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for algo in 1 3; do
for c in "0 0" "296 256"; do
  set -- $c
  timeout 300 $TR tools/phase_probe.py --ctas $1 --threads $2 --algo $algo 2>&1 | grep rank
done
done
for algo in 1 3; do
timeout 600 $TR bench.py --gpus $NP --no-e2e --algo $algo > gpurun_out/bench_n${NP}_a$algo.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_n${NP}_a$algo.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ['t_us','busbw_gbs','allreduce_only','nccl_allreduce_flat','easgd']})"
done
