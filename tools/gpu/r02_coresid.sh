# does a small-CTA NVLS allreduce run beside cuBLAS GEMMs? (tools/overlap_probe.py, p = 4)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
mkdir -p gpurun_out
for env in "THREADS=128 CTAS=148,296" "THREADS=128 CTAS=148,296 PRIO=1" "THREADS=512 CTAS=32,148" "THREADS=64 CTAS=296 PRIO=1"; do
  env GEMM_ONLY=1 NO_CARVEOUT=1 SYM=1 ALGO=4 $env timeout 300 $TR --master-port 29594 tools/overlap_probe.py 2>/dev/null | grep "p=" | sed "s/^/[$env] /" | tee -a gpurun_out/coresid.txt
done
timeout 300 env GEMM_ONLY=1 NO_CARVEOUT=1 CTAS=32,148 $TR --master-port 29595 tools/overlap_probe.py 2>/dev/null | grep "p=" | sed "s/^/[tma] /" | tee -a gpurun_out/coresid.txt
