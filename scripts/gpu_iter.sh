# Iteration loop: GPU tests, p=1 local-kernel variants, p=NP phase timings per TC_VARIANT.
export TC_TIMEOUT_MS=10000
NP=${NP:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 29512"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/local_variants.py 2>&1 | head -2
for v in ${VARIANTS:-0 1}; do
for algo in 1 3; do
  TC_VARIANT=$v timeout 300 $TR tools/phase_probe.py --algo $algo 2>&1 | grep rank | sed "s/^/v$v /"
done
done
