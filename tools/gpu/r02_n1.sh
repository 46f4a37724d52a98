mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x --durations=20 > gpurun_out/gputest_r02b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_r02b.log
python bench.py > gpurun_out/bench_r02_n1.json 2> gpurun_out/bench_r02_n1.err; echo "bench rc=$?"
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_r02_ref_n1.json 2> gpurun_out/bench_r02_ref_n1.err; echo "ref rc=$?"
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_n1.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_local_tma -s 3 -c 1 -o gpurun_out/r02_k_local_tma python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
tail -3 gpurun_out/gputest_r02b.log
