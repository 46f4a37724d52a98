export TC_TIMEOUT_MS=60000
mkdir -p gpurun_out/r01k
timeout 300 python tools/emulated_step.py 2 0 3 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_twoshot_tma -s 1 -c 1 -o gpurun_out/r01k/prof_twoshot_tma_p2_emulated python tools/emulated_step.py 2 0 3 > gpurun_out/r01k/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/r01k/prof_twoshot_tma_p2_emulated.ncu-rep --page raw --csv > gpurun_out/r01k/ncu_raw.csv 2>/dev/null; echo "export rc=$?"
timeout 900 compute-sanitizer --tool memcheck --leak-check no python -m pytest tests/test_gpu_parity.py -x -q -k "unaligned or esgd or tile_boundaries or mixed_alignment" > gpurun_out/r01k/memcheck.log 2>&1; echo "memcheck rc=$?"
tail -5 gpurun_out/r01k/memcheck.log
