for L in libtc libtc_l1 libtc_l2 libtc_l3 libtc_l4; do
echo "== $L"
TC_LIB=$PWD/paper_1801_03855_b200/$L.so timeout 300 python tools/local_tma_ctas.py resnet50
done
