# one-shot without staging: real-process parity, then latency vs the other small-group paths
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -s > gpurun_out/mp_direct.log 2>&1; echo "mp rc=$?"; tail -1 gpurun_out/mp_direct.log
for N in 2 4; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 900 $TR --nproc-per-node $N --master-port 2957$N tools/latency_probe.py > gpurun_out/lat_direct_p$N.jsonl 2>/dev/null; echo "lat$N rc=$?"
  cat gpurun_out/lat_direct_p$N.jsonl
done
