export TC_TIMEOUT_MS=20000
for rep in 1 2 3; do
for L in libtc libtc_m128; do
TC_LIB=$PWD/paper_1801_03855_b200/$L.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2984$rep bench.py --gpus 4 --steps 300 --no-e2e --no-nccl 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L rep$rep N4', round(d['t_us'],1), 'ar', round(d['allreduce_only']['t_us'],1), 'easgd', round(d['easgd']['t_us'],1), 'cfg4', round(d['config4']['mean_step_us'],1))"
done
done
