"""Summarise an ncu report (or a --metrics launch-list CSV) into markdown for profiles/."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]
STALLS = ["long_scoreboard", "wait", "barrier", "short_scoreboard", "math_pipe_throttle",
          "no_instructions", "selected", "not_selected", "membar", "lg_throttle",
          "mio_throttle", "branch_resolving", "dispatch_stall"]


def from_report(path):
    if path.endswith("_raw.csv"):   # `ncu -i <rep> --page raw --csv` exported on the GPU box
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = [f"# ncu summary: {path}", ""]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        out.append(f"## {d.get('Kernel Name', '?')[:90]}")
        out.append("")
        out.append("| metric | value |")
        out.append("|---|---|")
        for k, name in KEYS:
            if k in d:
                out.append(f"| {name} (`{k}`) | {d[k]} {u.get(k, '')} |")
        st = []
        for s in STALLS:
            k = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if k in d and d[k] not in ("", "0"):
                st.append((int(float(d[k])), s))
        tot = sum(v for v, _ in st) or 1
        out.append("")
        out.append("warp-state samples: " + ", ".join(f"{s} {100.0 * v / tot:.0f}%"
                                                        for v, s in sorted(st, reverse=True)[:6]))
        out.append("")
    return "\n".join(out)


def from_launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    agg = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0][-60:]
        t = float(d["Metric Value"])
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += t
    tot = sum(v[1] for v in agg.values()) or 1.0
    out = [f"# launch list summary: {path}", "", "| kernel | launches | total ns | share |",
           "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| {k} | {n} | {t:.0f} | {100.0 * t / tot:.1f}% |")
    return "\n".join(out)


if __name__ == "__main__":
    p = sys.argv[1]
    print(from_launches(p) if p.endswith(".csv") and not p.endswith("_raw.csv")
          else from_report(p))
