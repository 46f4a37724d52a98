# f1 at small batches: p = 2 CTA budgets, and eager (no graph) at p = 4 with BucketedStep's defaults
mkdir -p gpurun_out
summ() { python -c "
import sys,json
for l in sys.stdin:
    if not l.startswith('{'): continue
    d=json.loads(l); print(d['n_gpus'], d['batch_per_gpu'], d['graph'], d.get('mode'), d.get('ctas'), d.get('side_stream_priority'), 'c/s/o', round(d['t_compute_us']), round(d['t_serial_us']), round(d['t_overlap_us']), 'step', round(d['t_step_alone_us']), 'hidden', round(d['hidden_fraction'],2), d['replicas_identical'])"; }
for c in 16 24 32; do for b in 8 4; do
  CUDA_VISIBLE_DEVICES=0,1 timeout 600 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2 --master-port 29603 bench_train.py --graph --channels-last --priority --batch $b --ctas $c 2>>gpurun_out/trs4.err | tee -a gpurun_out/train_small4.jsonl | summ
done; done
for b in 8 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4 --master-port 29604 bench_train.py --channels-last --priority --batch $b --ctas 48 2>>gpurun_out/trs4.err | tee -a gpurun_out/train_small4.jsonl | summ
done
