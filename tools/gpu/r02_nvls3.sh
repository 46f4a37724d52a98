# NVLS: parity of the claimed-tile allreduce build, then variant timings
mkdir -p gpurun_out
TC_LIB=tools/bin/var/libtc_claim.so timeout 600 python -m pytest tests/test_gpu_multiproc.py -q -x -s > gpurun_out/mp_claim.log 2>&1; echo "mp claim rc=$?"; tail -1 gpurun_out/mp_claim.log
VARIANTS="default claim s1024 s512rw3" bash tools/gpu/r02_nvls2.sh
