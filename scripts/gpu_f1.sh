export TC_TIMEOUT_MS=20000
timeout 900 python -m pytest tests/test_gpu_bucketed.py -x -q 2>&1 | tail -2
bash scripts/gpu_overlap2.sh 2>&1 | grep -v "rc=0"
