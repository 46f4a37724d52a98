export TC_TIMEOUT_MS=20000
CUDA_VISIBLE_DEVICES=0,1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29692 bench.py --gpus 2 --steps 100 --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N2', d['t_us'], d['allreduce_only']['t_us'], d['nccl_allreduce_flat']['t_us'])"
