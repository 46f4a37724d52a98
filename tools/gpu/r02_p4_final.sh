# round-2 multi-GPU evidence on the final build: parity over real processes, bench lines at
# N = 2 / 4, NVLink counters around a step-only bench, phase stamps
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -s > gpurun_out/mp_final.log 2>&1; echo "mp rc=$?"
for N in 2 4; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 600 $TR --nproc-per-node $N --master-port 2953$N bench.py --gpus $N > gpurun_out/bench_final_n$N.json 2> gpurun_out/bench_final_n$N.err; echo "bench$N rc=$?"
done
nvidia-smi nvlink -h > gpurun_out/nvlink_help.txt 2>&1; nvidia-smi nvlink -gt d > gpurun_out/nvlink_gt.txt 2>&1; echo "smi rc=$?"; head -20 gpurun_out/nvlink_gt.txt
for N in 2 4; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 600 python tools/nvlink_counters.py --steps 210 -- $TR --nproc-per-node $N --master-port 2955$N bench.py --gpus $N --steps 200 --warmup 10 --no-extras --no-e2e > gpurun_out/nvlink_n$N.txt 2> gpurun_out/nvlink_n$N.err; echo "nvl$N rc=$?"; tail -2 gpurun_out/nvlink_n$N.txt | cut -c1-1500
done
