# Multi-GPU evidence of the build in the tree (gpurun --gpus 4): real-process parity, bench lines
# and reference arms at N = 2 / 4, configs 3, config-5 sweeps
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -s > gpurun_out/ev_mp.log 2>&1; echo "mp rc=$?"; tail -1 gpurun_out/ev_mp.log
for N in 2 4; do
  V=$(seq -s, 0 $((N-1)))
  CUDA_VISIBLE_DEVICES=$V timeout 600 $TR --nproc-per-node $N --master-port 2953$N bench.py --gpus $N > gpurun_out/ev_bench_n$N.json 2> gpurun_out/ev_bench_n$N.err; echo "bench$N rc=$?"
  CUDA_VISIBLE_DEVICES=$V timeout 600 $TR --nproc-per-node $N --master-port 2954$N bench.py --gpus $N --impl reference --steps 5 --warmup 3 > gpurun_out/ev_ref_n$N.json 2>/dev/null; echo "ref$N rc=$?"
  for c in alexnet vgg16; do CUDA_VISIBLE_DEVICES=$V timeout 600 $TR --nproc-per-node $N --master-port 2955$N bench.py --gpus $N --config $c --steps 50 --no-e2e > gpurun_out/ev_bench_${c}_n$N.json 2>/dev/null; echo "$c$N rc=$?"; done
  if [ -n "$SWEEP" ]; then CUDA_VISIBLE_DEVICES=$V timeout 900 $TR --nproc-per-node $N --master-port 2956$N bench_sweep.py > gpurun_out/ev_sweep_p$N.jsonl 2>/dev/null; echo "sweep$N rc=$?"; fi
done
