export TC_TIMEOUT_MS=20000
mkdir -p gpurun_out/r01e
for NP in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 2959$NP"
CV=$([ $NP = 2 ] && echo 0,1 || echo 0,1,2,3)
: > gpurun_out/r01e/overlap8_p$NP.log
for args in "--compute gemm --bucket-mb 64" "--compute gemm --bucket-mb 48" "--compute gemm --bucket-mb 64 --ratio 2"; do
CUDA_VISIBLE_DEVICES=$CV timeout 600 $TR bench_overlap.py $args >> gpurun_out/r01e/overlap8_p$NP.log 2>&1; echo "overlap p$NP $args rc=$?"
done
grep bench gpurun_out/r01e/overlap8_p$NP.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['n_gpus'], d['compute'], d['mode'], d['bucket_mb'], d['ratio'], d['ctas'], 'comp_c', round(d['t_compute_carveout_us']), 'step', round(d['t_step_us']), 'compute', round(d['t_compute_us']), 'serial', round(d['t_serial_us']), 'overlap', round(d['t_overlap_us']), 'hidden', round(d['hidden_fraction'],2))"
done
