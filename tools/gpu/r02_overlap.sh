# NEXT row f1 at p = 4: high-priority side stream, with and without the GEMM SM carveout
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
show() { grep '^{' $1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$2', d['algo'], d['ctas'], d['mode'], d['sm_carveout'], round(d['t_step_us']), round(d['t_compute_us']), round(d['t_compute_carveout_us']), round(d['t_serial_us']), round(d['t_overlap_us']), round(d['hidden_fraction'],2))"; }
i=0
for cfg in "--priority --shapes 64,32,16" "--priority --carveout --shapes 64,32,16" "--priority --ratio 2 --shapes 64,32"; do
  i=$((i+1))
  timeout 300 $TR --master-port 2963$i bench_overlap.py --compute gemm $cfg > gpurun_out/overlap_p$i.jsonl 2> gpurun_out/overlap_p$i.err; echo "cfg$i rc=$?"; show gpurun_out/overlap_p$i.jsonl "p$i"
done
