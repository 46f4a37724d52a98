export TC_TIMEOUT_MS=20000
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for NP in 2 4; do
CV=$([ $NP = 2 ] && echo 0,1 || echo 0,1,2,3)
CUDA_VISIBLE_DEVICES=$CV timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 2979$NP bench.py --gpus $NP --steps 100 --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N$NP', round(d['t_us'],1), 'ar', round(d['allreduce_only']['t_us'],1), 'bcast', d['broadcast'])"
done
