"""Summarise ncu outputs into markdown for profiles/.

    python tools/profile_summary.py launches <launches.csv>            # per-kernel share of device time
    python tools/profile_summary.py full <report.ncu-rep> [kernel...]  # key metrics + stall reasons
"""
import collections
import csv
import json
import subprocess
import sys

_UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def launches(path):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for row in csv.DictReader(lines):
        if row.get("Metric Name") != "gpu__time_duration.sum":
            continue
        us = float(row["Metric Value"].replace(",", "")) * _UNIT.get(row["Metric Unit"], 1.0)
        name = row["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total (ms) | share | avg (us) |", "|---|---|---|---|---|"]
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {n} | {us / 1e3:.2f} | {100 * us / tot:.1f}% | {us / n:.1f} |")
    out.append(f"| **total** | {sum(v[0] for v in agg.values())} | {tot / 1e3:.2f} | 100% | |")
    return "\n".join(out)


def _num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return None


def full(rep, kernels=()):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(raw.splitlines())
    hdr = next(r)
    units = dict(zip(hdr, next(r)))
    rows = []
    for row in r:
        d = dict(zip(hdr, row))
        name = d["Kernel Name"]
        if kernels and not any(k in name for k in kernels):
            continue
        stalls = [(_num(v), h.replace("smsp__pcsamp_warps_issue_stalled_", "")) for h, v in d.items()
                  if "smsp__pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued") and _num(v) is not None]
        tot = sum(v for v, _ in stalls) or 1.0
        top = ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(stalls, reverse=True)[:5])
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
        dram = sum((_num(d.get(k, 0)) or 0) * scale.get(units.get(k, "Mbyte"), 1.0)
                   for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        dram_unit = "Mbyte"
        rows.append({
            "kernel": name.split("(")[0],
            "duration_us": _num(d.get("gpu__time_duration.sum")),
            "duration_unit": units.get("gpu__time_duration.sum"),
            "issue_active_pct": _num(d.get("sm__inst_issued.avg.pct_of_peak_sustained_active")),
            "warps_active_pct": _num(d.get("sm__warps_active.avg.pct_of_peak_sustained_active")),
            "ipc": _num(d.get("sm__inst_executed.avg.per_cycle_active")),
            "registers": _num(d.get("launch__registers_per_thread")),
            "grid": _num(d.get("launch__grid_size")),
            "block": _num(d.get("launch__block_size")),
            "dram_bytes": dram, "dram_unit": dram_unit,
            "l2_hit_pct": _num(d.get("lts__t_sector_hit_rate.pct")),
            "fma_pipe_pct": _num(d.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active")),
            "alu_pipe_pct": _num(d.get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active")),
            "top_stalls": top,
        })
    out = ["| kernel | dur | issue % | warps active % | IPC | regs | grid x block | DRAM r+w | L2 hit % | FMA/ALU pipe % | top stalls |",
           "|---|---|---|---|---|---|---|---|---|---|---|"]
    for x in rows:
        out.append(f"| `{x['kernel']}` | {x['duration_us']} {x['duration_unit']} | {x['issue_active_pct']:.1f} | "
                   f"{x['warps_active_pct']:.1f} | {x['ipc']:.2f} | {x['registers']:.0f} | {x['grid']:.0f}x{x['block']:.0f} | "
                   f"{x['dram_bytes']:.1f} {x['dram_unit']} | {x['l2_hit_pct']:.1f} | {x['fma_pipe_pct']:.1f}/{x['alu_pipe_pct']:.1f} | {x['top_stalls']} |")
    return "\n".join(out), rows


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    else:
        md, rows = full(sys.argv[2], sys.argv[3:])
        print(md)
        print(json.dumps(rows))
