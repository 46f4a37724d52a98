# round-2 multi-GPU session: real-process parity, bench lines at N = 2 / 4, phase stamps
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -s > gpurun_out/mp_r02.log 2>&1; echo "mp rc=$?"
for N in 2 4; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 600 $TR --nproc-per-node $N --master-port 2953$N bench.py --gpus $N > gpurun_out/bench_r02_n$N.json 2> gpurun_out/bench_r02_n$N.err; echo "bench$N rc=$?"
done
for N in 2 4; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 300 $TR --nproc-per-node $N --master-port 2954$N tools/phase_probe.py --algo 6 --sym > gpurun_out/phase_r02_p$N.txt 2>&1; echo "phase$N rc=$?"
done
CUDA_VISIBLE_DEVICES=0,1 timeout 300 $TR --nproc-per-node 2 --master-port 29561 tools/nvl_probe.py > gpurun_out/nvl_probe_p2.jsonl 2> gpurun_out/nvl_probe_p2.err; echo "probe2 rc=$?"
