export TC_TIMEOUT_MS=20000
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29731"
for c in 0 37 74 148; do
timeout 300 $TR tools/phase_probe.py --numel 262144 --algo 0 --oneshot -1 --ctas $c --iters 50 2>&1 | grep "rank 0" | head -1 | cut -c1-200
done
for c in 16 32 64 148; do
timeout 300 $TR tools/phase_probe.py --numel 262144 --algo 6 --oneshot 0 --ctas $c --iters 50 2>&1 | grep "rank 0" | head -1 | cut -c1-200
done
