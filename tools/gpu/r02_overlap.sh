# NEXT row f1 at p = 4: bucketed step beside cuBLAS GEMMs -- TMA two-shot vs register pull whose
# CTAs (no shared memory) can share an SM with a GEMM CTA
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
show() { grep '^{' $1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$2', d['algo'], d['threads'], d['ctas'], d['mode'], round(d['t_step_us']), round(d['t_compute_us']), round(d['t_serial_us']), round(d['t_overlap_us']), round(d['hidden_fraction'],2))"; }
i=0
for cfg in "--algo 1 --threads 256 --shapes 148,296" "--algo 1 --threads 128 --shapes 148,296,592" "--algo 6 --shapes 16,8"; do
  i=$((i+1))
  timeout 300 $TR --master-port 2960$i bench_overlap.py --compute gemm $cfg > gpurun_out/overlap_c$i.jsonl 2> gpurun_out/overlap_c$i.err; echo "cfg$i rc=$?"; show gpurun_out/overlap_c$i.jsonl c$i
done
