export TC_TIMEOUT_MS=10000
NP=${NP:-4}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 29531"
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q 2>&1 | tail -2
for v in 0 3; do
  TC_VARIANT=$v timeout 300 $TR tools/phase_probe.py --sym --algo 4 2>&1 | grep -E "rank 0" | head -4
done
timeout 300 $TR tools/phase_probe.py --sym --algo 1 2>&1 | grep -E "rank 0" | head -4
