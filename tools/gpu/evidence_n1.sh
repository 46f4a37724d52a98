# Single-GPU evidence of the build in the tree (profiles/README.md names what each output became):
# GPU suite, smoke, bench N = 1 + reference arm, configs 3 at N = 1, ncu launch list and one full
# capture of the dominant kernel (each ncu pass only after its command exited 0 without ncu)
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/ev_gputests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/ev_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/ev_smoke.log
python bench.py > gpurun_out/ev_bench_n1.json 2> gpurun_out/ev_bench_n1.err; echo "bench rc=$?"
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ev_ref_n1.json 2> gpurun_out/ev_ref_n1.err; echo "ref rc=$?"
for c in alexnet vgg16; do python bench.py --config $c --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/ev_bench_${c}_n1.json 2>/dev/null; echo "$c rc=$?"; done
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_n1.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev_ncu1.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_local_tma -s 3 -c 1 -o gpurun_out/ev_k_local_tma python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev_ncu2.log 2>&1; echo "ncu2 rc=$?"
# the TMA two-shot (fused SGD) of p = 2 / 4 emulated ranks on this one GPU: DRAM bytes per launch
for P in 2 4; do
  python tools/emulated_step.py $P 6 3 > gpurun_out/ev_emu$P.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_twoshot_tma -s 1 -c 1 -o gpurun_out/ev_t2_emulated_p$P python tools/emulated_step.py $P 6 3 > gpurun_out/ev_ncu_t2_p$P.log 2>&1; echo "ncu t2 p$P rc=$?"
done
