"""Summarise an `ncu --set full` report of tools/profile_step.py into profiles/ncu_traffic.json.

usage: python tools/ncu_summary.py REPORT[,REPORT2...] "<source description>" [out.json]
One entry per kernel name (the first launch of each in the report); dram bytes are per launch.
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),  # ns -> us
    "dram_read_MB": ("dram__bytes_read.sum", 1e-6),
    "dram_write_MB": ("dram__bytes_write.sum", 1e-6),
    "registers": ("launch__registers_per_thread", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "tensor_pipe_active_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    "inst_executed": ("smsp__inst_executed.sum", 1),
    "l1_data_pipe_pct": ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", 1),
    "lts_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "issue_active_pct": ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", 1),
    # L1 data-pipe wavefronts by memory space (the shared-vs-global split of the LSU pipe)
    "l1_wavefronts_total_pct": ("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed", 1),
    "l1_wavefronts_shared_pct": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 1),
    "l1_wavefronts_shared": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3,
              "msecond": 1e6, "ms": 1e6}


def main():
    reps, source = sys.argv[1].split(","), sys.argv[2]
    out = sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_traffic.json"
    kernels = {}
    for rep in reps:
        summarise(rep, kernels)
    json.dump({"source": source, "report": " + ".join(reps) + " (not committed; summarised here)", "kernels": kernels},
              open(out, "w"), indent=1)
    print(json.dumps(kernels, indent=1))


def summarise(rep, kernels):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(head, r))
        name = d["Kernel Name"].split("(")[0].split("<")[0].split("::")[-1]  # template args dropped
        if name in kernels:
            continue
        e = {}
        for key, (metric, scale) in METRICS.items():
            if metric not in d or d[metric] in ("", "n/a", "no data"):
                continue
            u = units[head.index(metric)]
            v = float(d[metric].replace(",", "")) * UNIT_SCALE.get(u, 1)
            e[key] = round(v * scale, 3) if scale != 1 else v
        if "dram_read_MB" in e and "dram_write_MB" in e:
            e["dram_bytes"] = int(round((e["dram_read_MB"] + e["dram_write_MB"]) * 1e6))
        if e.get("l1_wavefronts_total_pct"):
            e["l1_wavefronts_shared_share"] = round(e.get("l1_wavefronts_shared_pct", 0.0) / e["l1_wavefronts_total_pct"], 3)
        kernels[name] = e


if __name__ == "__main__":
    main()
