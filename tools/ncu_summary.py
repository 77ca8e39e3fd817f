"""Summarise ncu reports (gpurun_out/*.ncu-rep) into profiles/ncu_summary.json
(per-launch DRAM traffic used by bench.py's roofline.traffic) and a markdown table."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
           "l1tex__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.sum",
           "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "byte": 1.0, "usecond": 1.0, "msecond": 1e3,
        "us": 1.0, "ms": 1e3}


def read(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = dict(zip(h, row))
        u = dict(zip(h, units))
        item = {"kernel": d.get("Kernel Name", "")[:120]}
        for m in METRICS:
            if m in d and d[m] not in ("", "n/a", "no data"):
                v = float(d[m].replace(",", ""))
                item[m] = v * UNIT.get(u.get(m, ""), 1.0)
        res.append(item)
    return res


def main():
    reps = [Path(p) for p in sys.argv[1:]]
    summary = {}
    lines = ["| report | kernel | time (us) | DRAM read+write (MB) | L2 bytes (MB) | fp64 pipe % | tensor pipe % | "
             "warps active % | regs |",
             "|---|---|---|---|---|---|---|---|---|"]
    for rep in reps:
        for it in read(rep):
            dram = it.get("dram__bytes_read.sum", 0) + it.get("dram__bytes_write.sum", 0)
            key = rep.stem.replace("prof_", "")
            key = key.split("_", 1)[1] if key[:1] == "r" and key[1:2].isdigit() else key  # r2_spmm -> spmm
            if "lts__t_sectors.sum" in it and "lts__t_bytes.sum" not in it:
                it["lts__t_bytes.sum"] = 32.0 * it["lts__t_sectors.sum"]
            summary[key] = {"kernel": it["kernel"], "dram_bytes_per_launch": dram,
                            "time_us": it.get("gpu__time_duration.sum"), **{k: v for k, v in it.items() if k != "kernel"}}
            lines.append(f"| {rep.name} | `{it['kernel'][:60]}` | {it.get('gpu__time_duration.sum', 0):.1f} | "
                         f"{dram / 1e6:.1f} | {it.get('lts__t_bytes.sum', 0) / 1e6:.1f} | "
                         f"{it.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                         f"{it.get('TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                         f"{it.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                         f"{it.get('launch__registers_per_thread', 0):.0f} |")
    print("\n".join(lines))
    return summary


if __name__ == "__main__":
    s = main()
    out = Path(__file__).resolve().parents[1] / "profiles" / "ncu_summary.json"
    old = json.loads(out.read_text()) if out.exists() else {}
    old.update(s)
    out.write_text(json.dumps(old, indent=1))
