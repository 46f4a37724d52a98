export TC_TIMEOUT_MS=20000
for L in libtc libtc_cw8u1 libtc_cw16u1 libtc_cw8u2; do
export TC_LIB=$PWD/paper_1801_03855_b200/$L.so
echo "== $L"
for NP in 2 4; do
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 2960$NP"
CV=$([ $NP = 2 ] && echo 0,1 || echo 0,1,2,3)
for c in 16 32 148; do
  CUDA_VISIBLE_DEVICES=$CV timeout 300 $TR tools/phase_probe.py --sym --algo 6 --ctas $c 2>&1 | grep -E "rank 0" | head -2 | sed 's/(busbw.*RS=/RS=/' | sed "s/^/p=$NP /"
done
done
done
