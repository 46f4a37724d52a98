# NVLS in-flight depth / grid sweep at p = 4 (allreduce and fused SGD), build variants
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
for v in default v1 v2 v3 v4; do
  if [ $v = default ]; then L=paper_1801_03855_b200/libtc.so; else L=tools/bin/var/libtc_$v.so; fi
  for c in 148 74 32; do
    TC_LIB=$L timeout 300 $TR --master-port 29582 tools/algo_bench.py --algos 4 --ops ar,sgd --steps 30 --ctas $c 2>/dev/null | grep '{' | sed "s/^/$v $c /" | tee -a gpurun_out/nv4.txt | cut -c1-260
  done
done
