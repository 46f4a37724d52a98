TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
for v in default bc2 bc8 bc16; do
  if [ $v = default ]; then L=paper_1801_03855_b200/libtc.so; else L=tools/bin/var/libtc_$v.so; fi
  TC_LIB=$L timeout 300 $TR --master-port 29591 tools/algo_bench.py --algos 0 --ops bc --steps 30 2>/dev/null | grep '{' | sed "s/^/$v /"
done
