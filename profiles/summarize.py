"""Summarise ncu output into the committed profiles/ evidence (run here, on the CPU box).

  python profiles/summarize.py launches gpurun_out/launches.csv            > profiles/rNN_launches.md
  python profiles/summarize.py full gpurun_out/prof_x.ncu-rep [label]      > profiles/rNN_x_ncu.md
"""
import collections
import csv
import io
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
    for r in data:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        cnt[name] += 1
    T = sum(tot.values())
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print("| `%s` | %d | %.3f | %.4f |" % (k, cnt[k], v, v / T))
    print("\n(ncu --metrics gpu__time_duration.sum --clock-control none: cold-cache, serialised launches; "
          "compare shares, not absolutes.)")


def full(path, label=""):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print("# ncu --set full: %s\n" % (label or path))
    for vals in rows[2:]:
        d = dict(zip(hdr, zip(units, vals)))
        print("## `%s`\n" % d.get("Kernel Name", ("", "?"))[1][:160])
        print("| metric | unit | value |\n|---|---|---|")
        for k in KEYS:
            if k in d:
                print("| %s | %s | %s |" % (k, d[k][0], d[k][1]))
        stalls = [(h, float(v[1])) for h, v in d.items() if re.match(r"smsp__pcsamp_warps_issue_stalled_\w+$", h)
                  and not h.endswith("not_issued") and v[1] not in ("", "n/a")]
        tot = sum(s for _, s in stalls) or 1.0
        print("\nPC-sampling stall reasons (share of samples):\n")
        for h, s in sorted(stalls, key=lambda x: -x[1])[:8]:
            print("- %s: %.1f%%" % (h.replace("smsp__pcsamp_warps_issue_stalled_", ""), 100 * s / tot))
        print()


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
