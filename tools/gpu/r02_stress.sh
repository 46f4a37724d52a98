# multi-process stress: every call changes the data, algorithms rotate (tools/stress_mp.py)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
mkdir -p gpurun_out
for N in 4 2; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 600 $TR --nproc-per-node $N --master-port 2959$N tools/stress_mp.py ${ITERS:-3000} 2>&1 | grep -E "stress|Error|error" | tee -a gpurun_out/stress.txt
done
