# f1 synthetic backward with more compute per step and more buckets (p = 4)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
mkdir -p gpurun_out
summ() { python -c "
import sys,json
for l in sys.stdin:
    if not l.startswith('{'): continue
    d=json.loads(l); print(d['ratio'], d['buckets'], d.get('mode'), d.get('ctas'), d.get('threads'), d.get('algo'), 'c/s/o', round(d['t_compute_us']), round(d['t_serial_us']), round(d['t_overlap_us']), 'hidden', round(d['hidden_fraction'],2))"; }
for r in 4 2; do for b in 16 32; do
  timeout 600 $TR --master-port 29596 bench_overlap.py --sym --algo 4 --priority --threads 128 --shapes 148 --ratio $r --bucket-mb $b 2>>gpurun_out/f1r.err | tee -a gpurun_out/f1r.jsonl | summ
  timeout 600 $TR --master-port 29597 bench_overlap.py --priority --shapes 32,148 --ratio $r --bucket-mb $b 2>>gpurun_out/f1r.err | tee -a gpurun_out/f1r.jsonl | summ
done; done
