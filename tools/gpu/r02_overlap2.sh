# f1 regression check: round-1 snapshot vs HEAD, same box
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
(cd tools/bin/r1 && timeout 300 $TR --master-port 29601 bench_overlap.py --compute gemm > ../../../gpurun_out/overlap_r1.jsonl 2>/dev/null); echo "r1 rc=$?"
timeout 300 $TR --master-port 29602 bench_overlap.py --compute gemm > gpurun_out/overlap_head.jsonl 2>/dev/null; echo "head rc=$?"
for f in r1 head; do echo "== $f"; grep '^{' gpurun_out/overlap_$f.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['ctas'], d['mode'], round(d['t_step_us']), round(d['t_compute_us']), round(d['t_serial_us']), round(d['t_overlap_us']))"; done
