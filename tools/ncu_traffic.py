"""Write profiles/<tag>_ncu_traffic.json from `ncu --set full` captures of eager layer steps:
DRAM bytes (read + write) and PCIe read bytes per launch and per segment, per ABI call and
config, for bench.py's roofline "traffic" field.
usage: python tools/ncu_traffic.py <tag> c2=<rep>:<segments per launch> c3=<rep>:<segs> ...

Per ABI call: select = score_kernel + rank_kernel (kvd_select_resolve_fetch: top-k + resolve +
fetch; select_kernel / cand_kernel on the general and index paths), attn = attn_kernel (attention + LSE merge).
Averaged over the captured launches."""
import csv
import io
import json
import subprocess
import sys

CALLS = {"select": ("score_kernel", "rank_kernel", "select_kernel", "cand_kernel"), "attn": ("attn_kernel",)}
METRICS = ("dram__bytes_read.sum", "dram__bytes_write.sum", "pcie__read_bytes.sum")


def kernels(rep):
    txt = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          ",".join(METRICS)], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def val(r, m):
        if m not in h:
            return None
        i = h.index(m)
        return float(r[i].replace(",", "")) * scale.get(units[i], 1)
    out = []
    for r in rows[2:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("kvd::", "").split("<")[0]
        out.append((name, val(r, METRICS[0]) + val(r, METRICS[1]), val(r, METRICS[2])))
    return out


def link_bytes(csv_path):
    """Mean host-memory bytes read (syslts__d_sectors_fill_sysmem x 32 B) per rank_kernel launch
    of an ncu launch list (the fused miss gather's zero-copy reads over PCIe)."""
    sys.path.insert(0, "tools")
    import ncu_summary
    import contextlib
    import io as _io
    with contextlib.redirect_stdout(_io.StringIO()):
        rows = ncu_summary.summarise(csv_path)
    for name, n, avg, share, rd, wr, pr, pw, sy in rows:
        if name.endswith("rank_kernel"):
            return sy, n
    return None, 0


def main():
    tag = sys.argv[1]
    res = {}
    args = sys.argv[2:]
    links = []
    if "--link" in args:
        i = args.index("--link")
        links = args[i + 1:]
        args = args[:i]
    for a in args:
        cfg, spec = a.split("=", 1)
        rep, segs = spec.rsplit(":", 1)
        segs = int(segs)
        ks = kernels(rep)
        res[cfg] = {}
        for call, names in CALLS.items():
            per = {n: [(b, pc) for k, b, pc in ks if k == n] for n in names}
            per = {n: v for n, v in per.items() if v}
            if not per:
                continue
            first = next(iter(per))
            dram = sum(sum(b for b, _ in v) / len(v) for v in per.values() if v)
            pcie = [pc for v in per.values() for _, pc in v]
            pcie = sum(pcie) / len(per[first]) if pcie and None not in pcie else None
            res[cfg][call] = {"dram_bytes_per_launch": dram, "segments_per_launch": segs,
                              "dram_bytes_per_segment": dram / segs,
                              "pcie_read_bytes_per_launch": pcie,
                              "pcie_read_bytes_per_segment": None if pcie is None else pcie / segs,
                              "launches": len(per[first]),
                              "kernels": " + ".join(per) + f" ({rep.split('/')[-1]})"}
    for a in links:                                # host-link reads of the select call (launch list)
        cfg, spec = a.split("=", 1)
        csv_path, segs = spec.rsplit(":", 1)
        sy, n = link_bytes(csv_path)
        if sy is not None and cfg in res and "select" in res[cfg]:
            e = res[cfg]["select"]
            e["pcie_read_bytes_per_launch_source"] = f"syslts__d_sectors_fill_sysmem x 32 B, {n} rank_kernel launches " \
                                                     f"of {csv_path.split('/')[-1]} ({segs} segments each)"
            e["pcie_read_bytes_per_segment"] = sy / int(segs)
    path = f"profiles/{tag}_ncu_traffic.json"
    json.dump(res, open(path, "w"), indent=1)
    print(path, json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
