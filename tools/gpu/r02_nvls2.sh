# NVLS fused-SGD diagnosis at p = 4: phase stamps (default build) and build variants
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
timeout 300 $TR --master-port 29581 tools/phase_probe.py --algo 4 --sym > gpurun_out/phase_nvls_p4.txt 2>&1; echo "phase rc=$?"
for v in default r1 r2 r1w3; do
  if [ $v = default ]; then L=paper_1801_03855_b200/libtc.so; else L=tools/bin/var/libtc_$v.so; fi
  TC_LIB=$L timeout 300 $TR --master-port 29582 tools/algo_bench.py --algos 4 --ops ar,sgd --steps 30 > gpurun_out/nv_$v.jsonl 2>/dev/null; echo "$v rc=$?"
  sed "s/^/$v /" gpurun_out/nv_$v.jsonl
done
grep rank gpurun_out/phase_nvls_p4.txt
