"""Markdown table of a round's bench lines (DESIGN.md §12 / BASELINE.md §4).

    python tools/results_table.py gpurun_out/r02b_bench_*.json
"""
import json
import sys


def load(path):
    try:
        return json.loads(open(path).read().strip().splitlines()[-1])
    except Exception:                                        # noqa: BLE001
        return None


def main():
    rows = []
    for path in sys.argv[1:]:
        d = load(path)
        if not d or "roofline" not in d:
            continue
        c = d["config"]
        r = d["roofline"]
        iso = d.get("kernels_isolated") or {}
        k = d.get("kernels") or {}

        def iso_frac(kind):
            e = iso.get(kind)
            return f"{e['frac_hbm']:.2f}" if isinstance(e, dict) and "frac_hbm" in e else "—"

        def chained(kind):
            e = k.get(kind)
            return f"{e['avg_launch_us']:.1f}" if e else "—"
        name = c["workload"] + (f" α={c['alpha']:g}" if c.get("alpha") != 0.9 else "")
        rows.append((name, f"{d['value']:.0f}", f"{d['ms_per_step']:.3f}",
                     f"{(d.get('e2e') or {}).get('value', 0):.0f}", f"{d.get('hit_rate', 0):.3f}",
                     f"{r['bound']} {r['achieved']:.1f} {r['unit']} = **{r['frac']:.2f}**",
                     f"{d['hbm_step']['frac']:.2f}", iso_frac("score"), iso_frac("attn"),
                     f"{chained('score')} / {chained('select')} / {chained('attn')}", str(c.get("chains")),
                     f"{d['clocks'].get('sm_mhz')}"))
    print("| Config | tokens/s | ms/step | e2e tokens/s | hit rate | binding roofline (step) | HBM step frac | "
          "score kernel alone | attention alone | chained µs/launch score / rank / attn | chains | SM MHz |")
    print("|" + "---|" * 12)
    for r in rows:
        print("| " + " | ".join(r) + " |")


if __name__ == "__main__":
    main()
