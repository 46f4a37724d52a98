export TC_TIMEOUT_MS=20000
for NP in 2 4; do
CV=$([ $NP = 2 ] && echo 0,1 || echo 0,1,2,3)
CUDA_VISIBLE_DEVICES=$CV timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 2965$NP tools/phase_probe.py --sym --algo 6 --smid 2>&1 | grep -A2 "rank 0" | head -6
done
