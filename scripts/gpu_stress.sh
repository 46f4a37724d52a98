export TC_TIMEOUT_MS=20000
for NP in 2 4; do
CV=$([ $NP = 2 ] && echo 0,1 || echo 0,1,2,3)
CUDA_VISIBLE_DEVICES=$CV timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 2980$NP tools/stress_mp.py 5000 2>&1 | grep -E "stress|Error|error" | head -5
done
