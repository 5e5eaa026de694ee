"""Print key metrics and the hottest SASS lines (warp-stall samples) of kernels in an .ncu-rep."""
import csv
import io
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'Achieved Occupancy', 'Theoretical Occupancy',
        'Registers Per Thread', 'Waves Per SM', 'Compute (SM) Throughput', 'Grid Size', 'Block Size',
        'Eligible Warps Per Scheduler', 'Issued Warp Per Scheduler', 'No Eligible', 'L2 Hit Rate']


def ncu(*a):
    return subprocess.run(["ncu", "-i", *a], capture_output=True, text=True).stdout


def details(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    h = rows[0]
    ki, mi, vi, ui = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
    ii = h.index('ID')
    cur = None
    for r in rows[1:]:
        key = (r[ii], r[ki].split('(')[0])
        if key != cur:
            print('==', *key)
            cur = key
        if r[mi] in WANT:
            print('   ', r[mi], r[vi], r[ui])


def hot(rep, kernel, n=20):
    txt = ncu(rep, "--page", "source", "--csv", "-k", kernel, "--print-source", "sass")
    rows = list(csv.reader(io.StringIO(txt)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0] != "Address"]
    si, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    tot = sum(float(r[si] or 0) for r in data) or 1
    print(f"-- hottest SASS of {kernel} ({len(data)} instructions)")
    for r in sorted(data, key=lambda r: -float(r[si] or 0))[:n]:
        print(f"   {float(r[si]) / tot:6.3f}  {r[src][:100]}")


def stalls(rep, kernel):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv", "-k", kernel))))
    h, v = rows[0], rows[2]
    out = []
    for i, name in enumerate(h):
        if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
            try:
                out.append((float(v[i]), name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    print(f"-- stall reasons of {kernel} (warps per issue):", ", ".join(f"{n}={x:.2f}" for x, n in sorted(out, reverse=True)[:8]))


if __name__ == "__main__":
    rep = sys.argv[1]
    details(rep)
    for k in sys.argv[2:]:
        stalls(rep, k)
        hot(rep, k)


def by_line(rep, kernel, n=30):
    """Stall samples and executed instructions aggregated per CUDA source line."""
    txt = ncu(rep, "--page", "source", "--csv", "-k", kernel, "--print-source", "cuda,sass")
    rows = list(csv.reader(io.StringIO(txt)))
    out, fname, hdr = [], None, None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and fname and len(r) == len(hdr) and r[0].isdigit():
            si = hdr.index("Warp Stall Sampling (All Samples)")
            ei = hdr.index("Instructions Executed")
            try:
                s_, e_ = float(r[si] or 0), float(r[ei] or 0)
            except ValueError:
                continue
            if s_ or e_:
                out.append((s_, e_, fname, int(r[0]), r[1].strip()[:90]))
    tot = sum(x[0] for x in out) or 1
    print(f"-- {kernel}: stall samples by source line (top {n})")
    for s_, e_, f, ln, src in sorted(out, reverse=True)[:n]:
        print(f"   {s_ / tot:6.3f} {e_:10.0f}  {f}:{ln}  {src}")
