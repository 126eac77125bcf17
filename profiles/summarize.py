"""Summarise ncu output kept under profiles/.

  python profiles/summarize.py launches <launches.csv>       per-kernel share of the launch list
  python profiles/summarize.py full <report.ncu-rep> [...]   key metrics of a --set full capture

The launch list comes from `ncu --metrics gpu__time_duration.sum --clock-control none` (serialised,
cold-cache per launch), so only the kernels' shares are comparable with the bench's CUDA-event times.
"""
import csv
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1tex throughput % (active)"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 LSU data-pipe wavefronts %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "LSU wavefronts, shared/shuffle"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2->L1 bytes"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short scoreboard / issue"),
]


def launches(path):
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("unnamed>::", "").replace("void ", "")
        v = float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    print(f"{'kernel':60s} {'launches':>8s} {'total us':>12s} {'avg us':>10s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{k[:60]:60s} {cnt[k]:8d} {v:12.1f} {v / cnt[k]:10.2f} {100 * v / s:6.1f}%")


def full(paths):
    for rep in paths:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        hdr, units = rows[0], rows[1]
        idx = {h: i for i, h in enumerate(hdr)}
        for r in rows[2:]:
            print(f"### {r[idx['Kernel Name']].split('(')[0]}  ({rep.split('/')[-1]})")
            for key, label in KEYS:
                if key in idx:
                    print(f"  {label:38s} {r[idx[key]]:>16s} {units[idx[key]]}")
            stalls = []
            for h, i in idx.items():
                if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                    try:
                        v = float(r[i])
                    except ValueError:
                        continue
                    if v >= 0.05:
                        stalls.append((v, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            if stalls:
                print("  stalls per issue: " + ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)))
            for h in ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                      "smsp__issue_active.avg.pct_of_peak_sustained_active",
                      "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                      "l1tex__data_bank_conflicts_pipe_lsu.sum",
                      "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
                      "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
                      "l1tex__data_pipe_lsu_wavefronts_mem_lg.sum" if False else "l1tex__data_pipe_lsu_wavefronts.sum",
                      "lts__t_sectors_srcunit_tex_op_read.sum",
                      "dram__throughput.avg.pct_of_peak_sustained_elapsed"):
                if h in idx:
                    print(f"  {h:70s} {r[idx[h]]:>16s} {units[idx[h]]}")
            print()


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2:])
