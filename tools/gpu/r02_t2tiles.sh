TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  for v in default t256 t1024 smem224; do
    if [ $v = default ]; then L=paper_1801_03855_b200/libtc.so; else L=tools/bin/var/libtc_$v.so; fi
    CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) TC_LIB=$L timeout 300 $TR --nproc-per-node $N --master-port 2965$N tools/algo_bench.py --algos 6 --ops ar,sgd --steps 50 2>/dev/null | grep '{' | sed "s/^/$v /"
  done
done
