# two-shot with split (published-half) phases: parity on one GPU (emulated) and timings at p = 2 / 4
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
TC_LIB=tools/bin/var/libtc_split2.so CUDA_VISIBLE_DEVICES=0 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_graph.py tests/test_gpu_esgd.py -m gpu -q -x > gpurun_out/split_tests.log 2>&1; echo "split tests rc=$?"; tail -2 gpurun_out/split_tests.log
for N in 2 4; do
  for L in paper_1801_03855_b200/libtc.so tools/bin/var/libtc_split2.so; do
    CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) TC_LIB=$L timeout 300 $TR --nproc-per-node $N --master-port 2961$N tools/algo_bench.py --algos 6 --ops ar,sgd --steps 50 2>/dev/null | grep '{' | sed "s|^|$N $(basename $L) |"
  done
  CUDA_VISIBLE_DEVICES=$(seq -s, 0 $((N-1))) TC_LIB=tools/bin/var/libtc_split2.so timeout 300 $TR --nproc-per-node $N --master-port 2962$N tools/phase_probe.py --algo 6 --sym 2>&1 | grep "rank 0"
done
