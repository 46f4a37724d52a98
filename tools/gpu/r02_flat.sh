# flat one-shot + re-fitted LL limits: one-GPU parity, real-process parity, config-5 sweeps
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/flat_gpu_tests.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/flat_gpu_tests.log
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -s > gpurun_out/flat_mp.log 2>&1; echo "mp rc=$?"; tail -3 gpurun_out/flat_mp.log
for N in 4 2; do
  V=$(seq -s, 0 $((N-1)))
  CUDA_VISIBLE_DEVICES=$V timeout 900 $TR --nproc-per-node $N --master-port 2956$N bench_sweep.py > gpurun_out/flat_sweep_p$N.jsonl 2>gpurun_out/flat_sweep_p$N.err; echo "sweep$N rc=$?"
done
