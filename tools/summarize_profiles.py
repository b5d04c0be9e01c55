"""Summarise ncu outputs into profiles/ (tracked).

    python tools/summarize_profiles.py launches <launches.csv> <out.md>
    python tools/summarize_profiles.py report <file.ncu-rep> <out.md>
"""

import collections
import csv
import subprocess
import sys


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0.0, 0])
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0].replace("void ", "")
            agg[name][0] += float(r[vi].replace(",", ""))
            agg[name][1] += 1
    tot = sum(v[0] for v in agg.values())
    lines = [f"# ncu launch list: `{path}`", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none` over the whole bench command "
             "(cold-cache, serialised launches: compare shares, not absolutes).", "",
             f"Total kernel time {tot / 1e6:.1f} ms over {sum(v[1] for v in agg.values())} launches.", "",
             "| share | total ms | launches | kernel |", "|---:|---:|---:|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:30]:
        lines.append(f"| {v[0] / tot * 100:.1f}% | {v[0] / 1e6:.2f} | {v[1]} | `{k}` |")
    open(out, "w").write("\n".join(lines) + "\n")


WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
]


def report(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full: `{path}`", ""]
    for r in rows[2:]:
        kname = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines += [f"## `{kname[:120]}`", "", "| metric | value | unit |", "|---|---:|---|"]
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                lines.append(f"| {w} | {r[i]} | {units[i]} |")
        stalls = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), r[i]) for i, h in enumerate(hdr)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
        stalls = [(h, float(v)) for h, v in stalls if v.replace(".", "", 1).isdigit()]
        tot = sum(v for _, v in stalls) or 1.0
        lines += ["", "Warp stall samples (top 8):", ""]
        for h, v in sorted(stalls, key=lambda x: -x[1])[:8]:
            lines.append(f"* {h}: {v / tot * 100:.1f}%")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2], sys.argv[3])
