TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 4 2; do
  for v in default osflat; do
    if [ $v = default ]; then L=paper_1801_03855_b200/libtc.so; else L=tools/bin/var/libtc_$v.so; fi
    CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) TC_LIB=$L LAT_KIB=256,512,1024,2048,4096 timeout 300 $TR --nproc-per-node $N --master-port 2968$N tools/latency_probe.py 2>/dev/null | grep '{' | sed "s/^/$v /"
  done
done
