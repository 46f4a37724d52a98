export TC_TIMEOUT_MS=10000
NP=2
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 29531"
for a in 1 3; do
  for v in 0 1; do
  echo "algo=$a variant=$v"
  TC_VARIANT=$v timeout 300 $TR tools/phase_probe.py --sym --algo $a 2>&1 | grep -E "rank" | head -4
  done
done
timeout 300 $TR tools/phase_probe.py --algo 1 2>&1 | grep -E "rank" | head -4
