"""One-line summary of a bench.py JSON line (value, step, roofline, per-kernel timings)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:                                   # noqa: BLE001
        print(path, "unreadable:", e)
        continue
    if "impl" in d:
        print(path, d.get("impl"), round(d["value"], 2), d["unit"], "ms/step", round(d["ms_per_step"], 1))
        continue
    r = d["roofline"]
    ks = " ".join(f"{k}:{v['avg_launch_us']:.1f}us/{v.get('frac_hbm_per_launch', 0):.2f}x{v['launches_per_step']:.0f}"
                  for k, v in d["kernels"].items())
    print(f"{d['config']['workload']} {d['value']:.0f} tok/s {d['ms_per_step']:.3f} ms (timer {d.get('ms_per_step_with_kernel_timer') or 0:.3f})"
          f" hit {d['hit_rate']:.3f} roof {r['bound']} {r['frac']:.2f} hbm_step {d['hbm_step']['frac']:.2f} | {ks}"
          f" | e2e {(d.get('e2e') or {}).get('value', 0):.0f}"
          + (" | iso " + " ".join(f"{k}:{v['avg_launch_us']:.1f}us/{v['frac_hbm']:.2f}" for k, v in d["kernels_isolated"].items()
                                  if isinstance(v, dict)) if d.get("kernels_isolated") else ""))
