# f1 regression bisect, part 2
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
show() { grep '^{' $1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$2', d['ctas'], d['mode'], round(d['t_step_us']), round(d['t_compute_us']), round(d['t_serial_us']), round(d['t_overlap_us']))"; }
timeout 300 $TR --master-port 29604 tools/bin/bo_r1.py --compute gemm > gpurun_out/overlap_head_r1bo.jsonl 2>/dev/null; echo "head lib + r1 bench_overlap rc=$?"; show gpurun_out/overlap_head_r1bo.jsonl head_lib_r1bo
for w in w_4130056 w_802ebbe; do
  (cd tools/bin/$w && timeout 300 $TR --master-port 29603 bench_overlap.py --compute gemm > ../../../gpurun_out/overlap_$w.jsonl 2>/dev/null); echo "$w rc=$?"; show gpurun_out/overlap_$w.jsonl $w
done
