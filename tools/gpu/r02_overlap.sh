# NEXT row f1 at p = 4: bucketed step beside cuBLAS GEMMs, with and without a green context
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
for G in 32 16 48; do
  timeout 300 $TR --master-port 2959$((G % 10)) bench_overlap.py --compute gemm --green $G > gpurun_out/overlap_green$G.jsonl 2> gpurun_out/overlap_green$G.err; echo "green$G rc=$?"; cat gpurun_out/overlap_green$G.jsonl; tail -3 gpurun_out/overlap_green$G.err
done
timeout 300 $TR --master-port 29599 bench_overlap.py --compute gemm > gpurun_out/overlap_plain.jsonl 2> gpurun_out/overlap_plain.err; echo "plain rc=$?"; cat gpurun_out/overlap_plain.jsonl
