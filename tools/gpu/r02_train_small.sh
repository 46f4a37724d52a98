# f1 on a graph-captured ResNet-50 iteration at small per-GPU batches (SMs not saturated), p = 4
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
mkdir -p gpurun_out
summ() { python -c "
import sys,json
for l in sys.stdin:
    if not l.startswith('{'): continue
    d=json.loads(l); print(d['batch_per_gpu'], d['bucket_mb'], d['buckets'], d.get('mode'), d.get('ctas'), d.get('side_stream_priority'), d.get('switch'), 'c/s/o', round(d['t_compute_us']), round(d['t_serial_us']), round(d['t_overlap_us']), 'step', round(d['t_step_alone_us']), 'hidden', round(d['hidden_fraction'],2), d['replicas_identical'])"; }
for b in 8 16 32; do
  for args in "" "--priority" "--priority --ctas 64" "--switch --split --threads 128 --ctas 148 --priority"; do
    timeout 600 $TR --master-port 29598 bench_train.py --graph --channels-last --batch $b $args 2>>gpurun_out/trs.err | tee -a gpurun_out/train_small.jsonl | summ
  done
done
