# SGD ring cap 160 KiB (new default) vs 192 KiB (old): bench.py A/B at N = 2, 4; then parity
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 4 2; do
  for rep in 1 2 3; do
    for v in new old; do
      if [ $v = new ]; then L=paper_1801_03855_b200/libtc.so; else L=tools/bin/var/libtc_old.so; fi
      CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) TC_LIB=$L timeout 300 $TR --nproc-per-node $N --master-port 2954$N bench.py --gpus $N --no-extras --no-e2e --no-cpu-baseline 2>/dev/null | grep '{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('$v', $N, round(d['t_us'],1), d['launch']['algo'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" | tee -a gpurun_out/ring_ab.txt
    done
  done
done
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/ring_gpu_tests.log 2>&1; echo "gpu rc=$?"; tail -2 gpurun_out/ring_gpu_tests.log
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -s > gpurun_out/ring_mp.log 2>&1; echo "mp rc=$?"; tail -2 gpurun_out/ring_mp.log
