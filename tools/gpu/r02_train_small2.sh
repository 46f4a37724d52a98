# f1 at small per-GPU batches: CTA budget / bucket size / split sweep (graph-captured, p = 4)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
mkdir -p gpurun_out
summ() { python -c "
import sys,json
for l in sys.stdin:
    if not l.startswith('{'): continue
    d=json.loads(l); print(d['batch_per_gpu'], d['bucket_mb'], d['buckets'], d.get('mode'), d.get('ctas'), d.get('side_stream_priority'), 'c/s/o', round(d['t_compute_us']), round(d['t_serial_us']), round(d['t_overlap_us']), 'step', round(d['t_step_alone_us']), 'hidden', round(d['hidden_fraction'],2), d['replicas_identical'])"; }
for b in 8 4; do
  for args in "--ctas 32" "--ctas 48" "--ctas 64" "--ctas 96" "--ctas 64 --bucket-mb 8" "--ctas 64 --bucket-mb 64" "--ctas 32 --split" "--ctas 64 --split"; do
    timeout 600 $TR --master-port 29599 bench_train.py --graph --channels-last --priority --batch $b $args 2>>gpurun_out/trs2.err | tee -a gpurun_out/train_small2.jsonl | summ
  done
done
