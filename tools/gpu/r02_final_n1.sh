# round-2 single-GPU evidence on the final build: GPU suite, smoke, bench N = 1 + reference arm,
# ncu launch list and one full capture of the dominant kernel
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/final_gputests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/final_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final_smoke.log
python bench.py > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.err; echo "bench rc=$?"
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final_ref_n1.json 2> gpurun_out/final_ref_n1.err; echo "ref rc=$?"
for c in alexnet vgg16; do python bench.py --config $c --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/final_bench_${c}_n1.json 2>/dev/null; echo "$c rc=$?"; done
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_n1.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_local_tma -s 3 -c 1 -o gpurun_out/final_k_local_tma python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
