# NEXT row f1 at p = 4: bucketed step beside cuBLAS GEMMs, plain and with green contexts
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
show() { grep '^{' $1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$2', d['ctas'], d['mode'], round(d['t_step_us']), round(d['t_compute_us']), round(d['t_serial_us']), round(d['t_overlap_us']), round(d['hidden_fraction'],2))"; }
timeout 300 $TR --master-port 29599 bench_overlap.py --compute gemm > gpurun_out/overlap_plain.jsonl 2> gpurun_out/overlap_plain.err; echo "plain rc=$?"; show gpurun_out/overlap_plain.jsonl plain
for G in 32 48; do
  timeout 300 $TR --master-port 2959$((G % 10)) bench_overlap.py --compute gemm --green $G > gpurun_out/overlap_green$G.jsonl 2> gpurun_out/overlap_green$G.err; echo "green$G rc=$?"; show gpurun_out/overlap_green$G.jsonl green$G; grep -i error gpurun_out/overlap_green$G.err | head -3
done
