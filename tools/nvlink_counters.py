"""NVLink byte counters around a command (diagnostics: the N >= 2 `traffic` evidence).

    python tools/nvlink_counters.py --steps K -- <command ...>

Reads `nvidia-smi nvlink -gt d` (per-link data TX/RX counters, KiB) for every visible GPU before
and after the command, and prints per GPU the TX/RX bytes moved and the bytes per step (the
command's K timed steps plus its warm-up, as given by --steps).  Not used inside bench.py: the
counters are read outside any timed region.
"""
import argparse
import json
import re
import subprocess
import sys


def read():
    out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d"], capture_output=True, text=True)
    gpus, cur = {}, None
    for line in out.stdout.splitlines():
        m = re.match(r"GPU (\d+):", line.strip())
        if m:
            cur = int(m.group(1))
            gpus[cur] = {"tx": 0, "rx": 0}
            continue
        m = re.search(r"Data (Tx|Rx):\s*([0-9]+)\s*KiB", line)
        if m and cur is not None:
            gpus[cur][m.group(1).lower()] += int(m.group(2)) * 1024
    return gpus, out.stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, required=True)
    ap.add_argument("cmd", nargs=argparse.REMAINDER)
    a = ap.parse_args()
    cmd = a.cmd[1:] if a.cmd and a.cmd[0] == "--" else a.cmd
    before, raw = read()
    if not before:
        print(json.dumps({"nvlink_counters": "unavailable", "nvidia_smi": raw[-500:]}))
        return
    r = subprocess.run(cmd)
    after, _ = read()
    res = {}
    for g in before:
        tx = after[g]["tx"] - before[g]["tx"]
        rx = after[g]["rx"] - before[g]["rx"]
        res[g] = {"tx_bytes": tx, "rx_bytes": rx, "tx_per_step": tx / a.steps,
                  "rx_per_step": rx / a.steps}
    print(json.dumps({"nvlink_counters": res, "steps": a.steps, "rc": r.returncode}), flush=True)
    sys.exit(r.returncode)


if __name__ == "__main__":
    main()
