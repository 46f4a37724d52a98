export TC_TIMEOUT_MS=20000
S=$(date +%s); timeout 900 python bench.py > /tmp/b1.log 2>&1; echo rc=$? wall=$(( $(date +%s) - S ))s
tail -1 /tmp/b1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N1', round(d['t_us'],1), d['roofline']['frac'], d['clocks'], d['steps'], d['gpu_launches'])"
S=$(date +%s); timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29830 bench.py --gpus 4 > /tmp/b4.log 2>&1; echo rc=$? wall=$(( $(date +%s) - S ))s
tail -1 /tmp/b4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N4', round(d['t_us'],1), d['roofline']['frac'], d['clocks'], d['allreduce_only']['t_us'])"
