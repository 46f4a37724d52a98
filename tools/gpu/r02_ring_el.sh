# stage-ring cap for the elastic ops (EASGD, fused elastic + SGD, async EASGD): bench.py extras A/B
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out
for N in 2 4; do for rep in 1 2; do for v in default el160 el128; do
  if [ $v = default ]; then L=paper_1801_03855_b200/libtc.so; else L=tools/bin/var/libtc_$v.so; fi
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) TC_LIB=$L timeout 300 $TR --nproc-per-node $N --master-port 2958$N bench.py --gpus $N --no-e2e --no-cpu-baseline --no-nccl --steps 100 2>/dev/null | grep '{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('$v', $N, 'step', round(d['t_us'],1), 'ea', round(d['easgd']['t_us'],1), 'async', round(d['easgd_async']['t_us'],1), 'esgd', round(d['esgd_fused']['t_us'],1), 'c4', round(d['config4']['mean_step_us'],1))" | tee -a gpurun_out/ring_el.txt
done; done; done
