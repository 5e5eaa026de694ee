"""Write profiles/<tag>_ncu_traffic.json from `ncu --set full` captures of one eager layer step
(whole batch, one chain): DRAM bytes (read + write) per ABI call, per config, for bench.py's
roofline "traffic" field.  usage: python tools/ncu_traffic.py <tag> c2=<rep> c3=<rep> ...

Per ABI call: select = score_kernel (+ topk_kernel when unfused), attn = attn_kernel +
merge_kernel.  Averaged over the captured layers."""
import csv
import io
import json
import subprocess
import sys

SEGMENTS = {"c2": 64, "c3": 128, "c4": 16, "c5": 512}
CALLS = {"select": ("score_kernel", "topk_kernel"), "attn": ("attn_kernel", "merge_kernel")}


def kernels(rep):
    txt = subprocess.run(["/usr/local/cuda/bin/ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    ri, wi = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out = []
    for r in rows[2:]:
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0]
        b = float(r[ri]) * scale[units[ri]] + float(r[wi]) * scale[units[wi]]
        out.append((name, b))
    return out


def main():
    tag = sys.argv[1]
    res = {}
    for a in sys.argv[2:]:
        cfg, rep = a.split("=", 1)
        ks = kernels(rep)
        res[cfg] = {}
        for call, names in CALLS.items():
            per = {n: [b for k, b in ks if k == n] for n in names}
            if not per[names[0]]:
                continue
            tot = sum(sum(v) / len(v) for v in per.values() if v)
            res[cfg][call] = {"dram_bytes_per_call": tot, "segments": SEGMENTS[cfg],
                              "kernels": " + ".join(n for n in names if per[n]) + f" ({rep.split('/')[-1]})"}
    path = f"profiles/{tag}_ncu_traffic.json"
    json.dump(res, open(path, "w"), indent=1)
    print(path, json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
