# NVLS fused step: reduction-warp count variants (p = 4, algo_bench, two runs each)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
mkdir -p gpurun_out
for rep in 1 2; do for v in default rw6 rw8u2 rw6e8; do
  if [ $v = default ]; then L=paper_1801_03855_b200/libtc.so; else L=tools/bin/var/libtc_$v.so; fi
  TC_LIB=$L timeout 300 $TR --master-port 29605 tools/algo_bench.py --algos 4 --ops sgd --steps 40 2>/dev/null | grep '{' | sed "s/^/$v /" | tee -a gpurun_out/nvls_sgd.txt | cut -c1-160
done; done
