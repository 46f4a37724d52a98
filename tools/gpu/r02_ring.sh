# TMA two-shot stage-ring size / tile size variants at p = 2, 4 (allreduce, fused SGD, EASGD)
mkdir -p gpurun_out
for N in 4 2; do
  TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node $N"
  for rep in 1 2; do
  for v in default s128 s160 s224 t256; do
    if [ $v = default ]; then L=paper_1801_03855_b200/libtc.so; else L=tools/bin/var/libtc_$v.so; fi
    CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) TC_LIB=$L timeout 300 $TR --master-port 2958$N tools/algo_bench.py --algos 6 --ops ar,sgd,ea --steps 40 2>/dev/null | grep '{' | sed "s/^/$v /" | tee -a gpurun_out/ring.txt | python -c "
import sys,json
for l in sys.stdin:
    v,j=l.split(' ',1); d=json.loads(j); print(v, d['p'], d['op'], round(d['median_us'],1), round(d['mean_us'],1))"
  done; done
done
