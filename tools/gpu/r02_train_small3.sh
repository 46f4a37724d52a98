# f1 with BucketedStep's new defaults (48-CTA budget, 25 MiB buckets, highest-priority stream)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_bucketed.py -q -x 2>&1 | tail -1
summ() { python -c "
import sys,json
for l in sys.stdin:
    if not l.startswith('{'): continue
    d=json.loads(l); print(d['batch_per_gpu'], d['bucket_mb'], d['buckets'], d.get('mode'), d.get('ctas'), d.get('side_stream_priority'), 'c/s/o', round(d['t_compute_us']), round(d['t_serial_us']), round(d['t_overlap_us']), 'step', round(d['t_step_alone_us']), 'hidden', round(d['hidden_fraction'],2), d['replicas_identical'])"; }
for b in 8 4 16; do
  for args in "--ctas 48 --priority" "--ctas 48"; do
    timeout 600 $TR --master-port 29600 bench_train.py --graph --channels-last --batch $b $args 2>>gpurun_out/trs3.err | tee -a gpurun_out/train_small3.jsonl | summ
  done
done
timeout 600 $TR --master-port 29601 bench_train.py --graph --channels-last --batch 8 --ctas 48 --priority 2>>gpurun_out/trs3.err | tee -a gpurun_out/train_small3_n4rep.jsonl | summ
CUDA_VISIBLE_DEVICES=0,1 timeout 600 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2 --master-port 29602 bench_train.py --graph --channels-last --batch 8 --ctas 48 --priority 2>>gpurun_out/trs3.err | tee -a gpurun_out/train_small3.jsonl | summ
