export TC_TIMEOUT_MS=20000
for L in libtc_m96; do
export TC_LIB=$PWD/paper_1801_03855_b200/$L.so
for NP in 2 4; do
CV=$([ $NP = 2 ] && echo 0,1 || echo 0,1,2,3)
for c in 148 296; do
CUDA_VISIBLE_DEVICES=$CV timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NP --master-addr 127.0.0.1 --master-port 2978$NP tools/phase_probe.py --sym --algo 6 --ctas $c 2>&1 | grep -E "rank 0" | head -2 | sed 's/(busbw.*RS=/RS=/' | sed "s/^/$L p=$NP /" | cut -c1-110
done
done
done
