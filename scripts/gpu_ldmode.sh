export TC_TIMEOUT_MS=10000
for L in libtc libtc_ld1 libtc_ld2; do
  export TC_LIB=$PWD/paper_1801_03855_b200/$L.so
  echo "== $L"
  timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N1', round(d['t_us'],1), round(d['roofline']['frac'],3))"
  for NP in 2 4; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 2954$NP bench.py --gpus $NP --steps 50 --warmup 5 --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N$NP', 'sgd', round(d['t_us'],1), 'ar', round(d['allreduce_only']['t_us'],1), 'nccl', round(d['nccl_allreduce_flat']['t_us'],1), 'easgd', round(d['easgd']['t_us'],1))"
  done
done
