export TC_TIMEOUT_MS=20000
CUDA_VISIBLE_DEVICES=0,1,2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29833 bench.py --gpus 3 --steps 100 > /tmp/b3.log 2>&1; echo rc=$?
tail -1 /tmp/b3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N3', round(d['t_us'],1), round(d['roofline']['frac'],3), 'ar', d['allreduce_only'], 'nccl', d['nccl_allreduce_flat']['t_us'], 'easgd', d['easgd']['t_us'], d['easgd']['clients'], 'bcast', d['broadcast']['t_us'])"
CUDA_VISIBLE_DEVICES=0,1,2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29834 tests/mp_worker.py 2>&1 | tail -2
echo mp rc=$?
