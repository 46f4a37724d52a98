mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_multiproc.py -q -x -s > gpurun_out/mp_bcast.log 2>&1; echo "mp rc=$?"; tail -2 gpurun_out/mp_bcast.log
for N in 2 4; do
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) timeout 600 $TR --nproc-per-node $N --master-port 2971$N bench.py --gpus $N --steps 100 --no-cpu-baseline --no-e2e > gpurun_out/bench_bcast_n$N.json 2>/dev/null; echo "bench$N rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/bench_bcast_n$N.json')); print($N, d['t_us'], d['broadcast'], d['allreduce_only']['t_us'], d.get('sgd_step_nvls',{}).get('t_us'))"
done
