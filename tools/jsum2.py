"""Print µs per call, stats-kernel µs and value of bench JSON lines (paths as arguments)."""
import json
import sys

for p in sys.argv[1:]:
    try:
        a = json.loads(open(p).read().strip().splitlines()[-1])
        print(f"{p}: {a['ms_per_step'] * 1e3:8.2f} us/call  kernel {a['roofline']['kernel_us']:8.2f} us  "
              f"value {a['value']:.4g}  launches {a['gpu_launches']}")
    except Exception as e:  # noqa: BLE001
        print(p, "unreadable:", e)
