"""Summarise an ncu --csv launch list: per kernel count, mean duration, share, DRAM bytes."""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in data:
        agg[r[ki].split("(")[0].replace("kvd::", "").split("<")[0]][r[mi]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(m["gpu__time_duration.sum"]) for m in agg.values())
    out = []
    for n, m in agg.items():
        t = m["gpu__time_duration.sum"]
        rd = sum(m.get("dram__bytes_read.sum", [0])) / len(t)
        wr = sum(m.get("dram__bytes_write.sum", [0])) / len(t)
        pr = sum(m.get("pcie__read_bytes.sum", [0])) / len(t)
        pw = sum(m.get("pcie__write_bytes.sum", [0])) / len(t)
        sy = 32 * sum(m.get("syslts__d_sectors_fill_sysmem.sum", [0])) / len(t)   # host-memory reads
        avg = sum(t) / len(t)
        out.append((n, len(t), avg, sum(t) / tot, rd, wr, pr, pw, sy))
        print(f"  {n:16s} n={len(t):4d} avg={avg / 1e3:9.2f} us share={sum(t) / tot:.3f} "
              f"dram rd={rd / 1e6:8.2f} MB wr={wr / 1e6:7.2f} MB -> {(rd + wr) / avg:7.1f} GB/s"
              f"  pcie rd={pr / 1e6:7.2f} MB wr={pw / 1e6:6.2f} MB  sysmem rd={sy / 1e6:7.2f} MB -> {sy / avg:6.1f} GB/s")
    return out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        summarise(p)
