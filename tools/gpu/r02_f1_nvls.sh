# f1 with the bucket allreduces on the switch (NVLS on few SMs), p = 4
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
summ() { python -c "
import sys,json
for l in sys.stdin:
    if not l.startswith('{'): continue
    d=json.loads(l); print(d.get('mode'), d.get('ctas'), d.get('algo'), 'c/s/o', round(d['t_compute_us']), round(d['t_serial_us']), round(d['t_overlap_us']), 'hidden', round(d['hidden_fraction'],2), d.get('replicas_identical',''))"; }
timeout 600 $TR --master-port 29591 bench_overlap.py --sym --algo 4 --priority --shapes 32,74 2>gpurun_out/f1nv_ov.err | tee gpurun_out/f1nv_overlap.jsonl | summ
timeout 600 $TR --master-port 29592 bench_overlap.py --sym --algo 4 --priority --shapes 32,74 --ratio 2 2>>gpurun_out/f1nv_ov.err | tee -a gpurun_out/f1nv_overlap.jsonl | summ
for args in "--split --ctas 32 --priority" "--ctas 32 --priority" "--split --ctas 32" "--split --ctas 74 --priority"; do
  timeout 600 $TR --master-port 29593 bench_train.py --graph --channels-last --switch $args 2>>gpurun_out/f1nv_tr.err | tee -a gpurun_out/f1nv_train.jsonl | summ
done
