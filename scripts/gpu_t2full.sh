export TC_TIMEOUT_MS=20000
mkdir -p gpurun_out/r01e
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for NP in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 2958$NP"
CV=$([ $NP = 2 ] && echo 0,1 || echo 0,1,2,3)
CUDA_VISIBLE_DEVICES=$CV timeout 600 $TR bench.py --gpus $NP > gpurun_out/r01e/bench_n$NP.log 2>&1; echo "bench n$NP rc=$?"
tail -1 gpurun_out/r01e/bench_n$NP.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N$NP', 'sgd', round(d['t_us'],1), d['config']['algo'], 'ar', round(d['allreduce_only']['t_us'],1), d['allreduce_only']['algo'], 'nccl', round(d['nccl_allreduce_flat']['t_us'],1), 'easgd', round(d['easgd']['t_us'],1), d['easgd']['algo'], 'e2e', d['e2e']['value'])"
CUDA_VISIBLE_DEVICES=$CV timeout 600 $TR bench_overlap.py > gpurun_out/r01e/overlap_p$NP.log 2>&1; echo "overlap rc=$?"
grep bench gpurun_out/r01e/overlap_p$NP.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['ctas'], 'step', round(d['t_step_us']), 'compute', round(d['t_compute_us']), 'serial', round(d['t_serial_us']), 'overlap', round(d['t_overlap_us']), 'hidden', round(d['hidden_fraction'],2))"
done
