export TC_TIMEOUT_MS=20000
for L in libtc libtc_small; do
for NC in "" 1; do
echo "== $L no_carveout=$NC"
CUDA_VISIBLE_DEVICES=0,1,2,3 GEMM_ONLY=1 NO_CARVEOUT=$NC TC_LIB=$PWD/paper_1801_03855_b200/$L.so timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29741 tools/overlap_probe.py 2>&1 | grep "p="
done
done
