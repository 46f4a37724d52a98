export TC_TIMEOUT_MS=20000
mkdir -p gpurun_out/r01
for NP in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 2957$NP"
CV=$([ $NP = 2 ] && echo 0,1 || echo 0,1,2,3)
CUDA_VISIBLE_DEVICES=$CV timeout 900 $TR bench_sweep.py --algo 6 --oneshot 0 --ll 0 --sizes 4,5,6,7,8,9,10 --tensors 1,161 --out gpurun_out/r01/sweep_tma_p$NP.jsonl > /dev/null 2>&1; echo "sweep p$NP rc=$?"
for A in 1 6; do
CUDA_VISIBLE_DEVICES=$CV timeout 600 $TR bench.py --gpus $NP --algo $A --steps 100 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N$NP algo $A', 'sgd', round(d['t_us'],1), 'ar', round(d['allreduce_only']['t_us'],1), d['allreduce_only']['algo'], 'nccl', round(d['nccl_allreduce_flat']['t_us'],1), 'easgd', round(d['easgd']['t_us'],1), d['easgd']['algo'])"
done
done
