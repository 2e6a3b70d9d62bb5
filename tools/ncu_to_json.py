"""Distil the round's ncu captures into the small JSON files bench.py reads:

  python tools/ncu_to_json.py gpurun_out/r2_search_c2.ncu-rep gpurun_out/r2_query_c2.ncu-rep

-> profiles/search_sm_c2.json, profiles/search_traffic_c2.json, profiles/query_c2.json
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}


def raw(rep):
    """metric -> value in base units (bytes, milliseconds)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    d = {}
    for name, unit, val in zip(rows[0], rows[1], rows[2]):
        try:
            d[name] = float(val.replace(",", "")) * SCALE.get(unit, 1.0)
        except ValueError:
            d[name] = val
    return d


def num(d, k):
    return float(d[k])


def main(search_rep, query_rep, n=100_000_000):
    s = raw(search_rep)
    t_ms = num(s, "gpu__time_duration.sum")
    sm = {"kernel": s["Kernel Name"], "workload": "C2 100M u64 lambda=9 IC-C", "n_keys": n,
          "gpu_time_ms": t_ms,
          "issue_active_pct": num(s, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
          "alu_pipe_pct_elapsed": num(s, "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed"),
          "lsu_shared_wavefront_pct_elapsed": num(
              s, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
          "warp_instructions": num(s, "smsp__inst_executed.sum"),
          "shared_wavefronts": num(s, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
          "shared_bank_conflicts": num(s, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
          "warps_active_pct": num(s, "sm__warps_active.avg.pct_of_peak_sustained_active"),
          "icc_hit_pct": num(s, "sm__icc_request_hit_rate.pct"),
          "dram_bytes": num(s, "dram__bytes_read.sum") + num(s, "dram__bytes_write.sum"),
          "source": f"ncu --set full ({Path(search_rep).name})"}
    (ROOT / "profiles" / "search_sm_c2.json").write_text(json.dumps(sm, indent=1) + "\n")
    tr = {"kernel": s["Kernel Name"], "workload": sm["workload"],
          "bytes_per_launch": int(sm["dram_bytes"]), "dram_read": int(num(s, "dram__bytes_read.sum")),
          "dram_write": int(num(s, "dram__bytes_write.sum")), "source": sm["source"]}
    (ROOT / "profiles" / "search_traffic_c2.json").write_text(json.dumps(tr, indent=1) + "\n")
    print(json.dumps(sm, indent=1))
    q = raw(query_rep)
    dq = num(q, "dram__bytes_read.sum") + num(q, "dram__bytes_write.sum")
    qd = {"kernel": q["Kernel Name"], "workload": "C2 batched query of 100M u64 keys",
          "n_queries": n, "gpu_time_ms": num(q, "gpu__time_duration.sum"),
          "dram_bytes": dq, "dram_bytes_per_query": dq / n,
          "l2_hit_pct": num(q, "lts__t_sector_hit_rate.pct"),
          "issue_active_pct": num(q, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
          "source": f"ncu --set full ({Path(query_rep).name})"}
    (ROOT / "profiles" / "query_c2.json").write_text(json.dumps(qd, indent=1) + "\n")
    print(json.dumps(qd, indent=1))
    return sm, qd


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
