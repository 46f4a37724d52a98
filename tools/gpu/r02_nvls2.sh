# NVLS fused-SGD diagnosis at p = 4: per build variant, timings and phase stamps
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
for v in ${VARIANTS:-f1 f2 f1r1}; do
  if [ $v = default ]; then L=paper_1801_03855_b200/libtc.so; else L=tools/bin/var/libtc_$v.so; fi
  TC_LIB=$L timeout 300 $TR --master-port 29582 tools/algo_bench.py --algos 4 --ops ar,sgd --steps 30 > gpurun_out/nv_$v.jsonl 2>/dev/null; echo "$v rc=$?"
  sed "s/^/$v /" gpurun_out/nv_$v.jsonl | grep '{'
  TC_LIB=$L timeout 300 $TR --master-port 29581 tools/phase_probe.py --algo 4 --sym > gpurun_out/phase_nvls_$v.txt 2>&1
  grep "rank 0" gpurun_out/phase_nvls_$v.txt | sed "s/^/$v /"
done
