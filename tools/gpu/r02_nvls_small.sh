# NVLS allreduce on small CTAs (f1: CTAs that fit beside a compute kernel's CTA), p = 4
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -s > gpurun_out/nvs_mp.log 2>&1; echo "mp rc=$?"; tail -1 gpurun_out/nvs_mp.log
for thr in 512 256 128 64; do for c in 148 296; do
  timeout 300 $TR --master-port 29591 tools/algo_bench.py --algos 4 --ops ar --steps 30 --ctas $c --threads $thr 2>/dev/null | grep '{' | tee -a gpurun_out/nvs_ar.jsonl | cut -c1-200
done; done
summ() { python -c "
import sys,json
for l in sys.stdin:
    if not l.startswith('{'): continue
    d=json.loads(l); print(d.get('mode'), d.get('ctas'), d.get('threads'), d.get('algo'), 'c/s/o', round(d['t_compute_us']), round(d['t_serial_us']), round(d['t_overlap_us']), 'hidden', round(d['hidden_fraction'],2), d.get('replicas_identical',''))"; }
for thr in 128 64; do
  timeout 600 $TR --master-port 29592 bench_overlap.py --sym --algo 4 --priority --threads $thr --shapes 148,296 2>>gpurun_out/nvs.err | tee -a gpurun_out/nvs_overlap.jsonl | summ
done
for args in "--split --ctas 148 --threads 128 --priority" "--split --ctas 296 --threads 64 --priority" "--split --ctas 148 --threads 128"; do
  timeout 600 $TR --master-port 29593 bench_train.py --graph --channels-last --switch $args 2>>gpurun_out/nvs.err | tee -a gpurun_out/nvs_train.jsonl | summ
done
