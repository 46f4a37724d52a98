TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 4 2 3; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) LAT_KIB=128,256,512,1024,2048,4096 timeout 300 $TR --nproc-per-node $N --master-port 2968$N tools/latency_probe.py 2>/dev/null | grep '{'
done
