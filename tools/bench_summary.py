"""Print the key fields of bench.py JSON lines read from stdin (or a file)."""
import json
import sys

src = open(sys.argv[1]) if len(sys.argv) > 1 else sys.stdin
for line in src:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    keys = ["impl", "n_gpus", "value", "tokens_per_s_per_gpu", "ms_per_step", "step_roofline_frac", "exposed_comm_ms",
            "kernel_ms", "roofline", "clocks", "e2e", "gpu_launches", "comm"]
    print(json.dumps({k: d[k] for k in keys if k in d}, indent=None))
