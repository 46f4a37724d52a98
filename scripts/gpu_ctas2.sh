export TC_TIMEOUT_MS=10000
NP=2
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 29531"
for c in 16 32 64 148 296; do
  timeout 300 $TR tools/phase_probe.py --sym --algo 1 --ctas $c 2>&1 | grep -E "rank 0" | head -2
done
