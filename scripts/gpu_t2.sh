export TC_TIMEOUT_MS=10000
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531"
for c in 16 32 64 148; do
  CUDA_VISIBLE_DEVICES=0,1 timeout 300 $TR tools/phase_probe.py --sym --algo 6 --ctas $c 2>&1 | grep -E "rank 0" | head -2
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532"
for c in 32 64 148; do
  timeout 300 $TR tools/phase_probe.py --sym --algo 6 --ctas $c 2>&1 | grep -E "rank 0" | head -2
done
