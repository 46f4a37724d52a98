export TC_TIMEOUT_MS=20000
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
