export TC_TIMEOUT_MS=20000
for NP in 2 4; do
CV=$([ $NP = 2 ] && echo 0,1 || echo 0,1,2,3)
for A in 4; do
CUDA_VISIBLE_DEVICES=$CV timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 2982$NP tools/phase_probe.py --sym --algo $A 2>&1 | grep -E "rank 0" | head -2 | sed 's/(busbw.*RS=/RS=/' | sed "s/^/p=$NP /" | cut -c1-100
done
done
