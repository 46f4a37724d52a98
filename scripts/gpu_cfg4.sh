export TC_TIMEOUT_MS=20000
for NP in 2 4; do
CV=$([ $NP = 2 ] && echo 0,1 || echo 0,1,2,3)
CUDA_VISIBLE_DEVICES=$CV timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 2976$NP bench.py --gpus $NP --steps 50 --no-e2e > /tmp/b$NP.log 2>&1; echo rc=$?
tail -1 /tmp/b$NP.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N$NP', d['t_us'], d.get('config4'))" 2>&1 | tail -2
tail -3 /tmp/b$NP.log | grep -i error | head -3
done
