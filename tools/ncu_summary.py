"""Summarise ncu output into the small text files kept under profiles/.

    python tools/ncu_summary.py launches LAUNCHES.csv OUT.csv [--note TEXT]
    python tools/ncu_summary.py full REPORT.ncu-rep OUT.txt [--algo-bytes B | --algo-flops F]

`launches`: per-kernel launch count, total time and share from an
`ncu --metrics gpu__time_duration.sum --csv` launch list.
`full`: the headline counters of one `ncu --set full` capture (duration,
pipe utilisation, DRAM bytes read/written, L2 hit rate, stall breakdown), and
the algorithmic bytes or flops of that launch next to them when given.
"""
import argparse
import collections
import csv
import io
import re
import subprocess
import sys


def _rows(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    return list(csv.reader(io.StringIO("".join(lines))))


def launches(path, out, note):
    rows = _rows(path)
    h = rows[0]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[1:]:
        name = re.sub(r"\(.*", "", r[ik]).replace("bgp::", "")
        tot[name] += float(r[iv].replace(",", "")) / 1e6
        cnt[name] += 1
    all_ms = sum(tot.values())
    with open(out, "w") as f:
        if note:
            f.write(f"# {note}\n")
        f.write(f"# {sum(cnt.values())} launches, {all_ms:.1f} ms total kernel time "
                "(ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)\n")
        f.write("kernel,launches,total_ms,share_pct\n")
        for k, v in tot.most_common():
            f.write(f"{k},{cnt[k]},{v:.2f},{100 * v / all_ms:.2f}\n")
    print(open(out).read())


WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe % (active)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe % (active)"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "shared pipe %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def full(path, out, algo_bytes, algo_flops):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        lines.append(f"kernel: {d.get('Kernel Name', '?')[:120]}")
        for key, label in WANT:
            if key in d and d[key] != "":
                lines.append(f"  {label:28s} {d[key]} {u.get(key, '')}".rstrip())
        stalls = {k: float(v) for k, v in d.items()
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                  and v not in ("", "0")}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
        lines.append("  stalls (warps per issue): " + ", ".join(
            f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
            f"={v:.2f}" for k, v in top))
        dur = float(d.get("gpu__time_duration.sum", "0") or 0) * 1e-9
        rd = float(d.get("dram__bytes_read.sum", "0") or 0)
        wr = float(d.get("dram__bytes_write.sum", "0") or 0)
        lines.append(f"  traffic (read+write)        {rd + wr:.4e} B")
        if algo_bytes:
            lines.append(f"  algorithmic bytes           {algo_bytes:.4e} B  (traffic/algorithmic = "
                         f"{(rd + wr) / algo_bytes:.2f}); achieved {algo_bytes / dur / 1e9:.1f} GB/s")
        if algo_flops:
            lines.append(f"  algorithmic flops           {algo_flops:.4e}  achieved {algo_flops / dur / 1e12:.2f} TFLOP/s")
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary of {path.split('/')[-1]} (clock-control none)\n")
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["launches", "full"])
    ap.add_argument("inp")
    ap.add_argument("out")
    ap.add_argument("--note", default="")
    ap.add_argument("--algo-bytes", type=float, default=0.0)
    ap.add_argument("--algo-flops", type=float, default=0.0)
    a = ap.parse_args()
    if a.mode == "launches":
        launches(a.inp, a.out, a.note)
    else:
        full(a.inp, a.out, a.algo_bytes, a.algo_flops)


if __name__ == "__main__":
    sys.exit(main())
