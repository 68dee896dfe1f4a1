"""Summaries of ncu --set full captures for profiles/: key counters, stall mix and the DRAM
traffic file bench.py reads. usage: python tools/ncu_summary.py TAG  (reads gpurun_out/prof_TAG_<kernel>.ncu-rep)"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
KERNELS = ["oz_vgemm_kernel", "oz_slice_kernel", "pair_kr_kernel", "pair_kr_kernel_pw4", "mo_kernel", "chi_kernel",
           "walk_kernel"]
TRAFFIC_NAME = {"pair_kr_kernel_pw4": "pair_kr_kernel"}  # the file bench.py reads for the Kramers path
WANT = ["gpu__time_duration.sum", "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes.sum.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread", "launch__grid_size",
        "smsp__warps_active.avg.per_cycle_active"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def main(tag):
    lines, traffic = [], None
    for k in KERNELS:
        rep = ROOT / "gpurun_out" / f"prof_{tag}_{k}.ncu-rep"
        if not rep.exists():
            continue
        h, u, v = raw(rep)
        lines.append(f"== {k} ({rep.name}; ncu --set full --clock-control none --import-source on, one steady-state "
                     f"launch of python tools/prof_step.py cfg4 6 20)")
        vals = {}
        for n, uu, x in zip(h, u, v):
            if n in WANT:
                lines.append(f"  {n:75s} {x} {uu}")
                vals[n] = (x, uu)
        st = []
        for n, x in zip(h, v):
            if "pcsamp_warps_issue_stalled" in n and not n.endswith("not_issued"):
                try:
                    st.append((float(x.replace(",", "")), n))
                except ValueError:
                    pass
        tot = sum(a for a, _ in st) or 1.0
        lines.append("  stall mix: " + ", ".join(f"{n.replace('smsp__pcsamp_warps_issue_stalled_', '')} "
                                                 f"{a / tot * 100:.1f}%" for a, n in sorted(st, reverse=True)[:6]))
        num = lambda n: float(vals[n][0].replace(",", "")) * SCALE.get(vals[n][1], 1.0)  # noqa: E731
        r, w = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
        notes = {"pair_kr_kernel_pw4": "O-only pass of the INT8 path: reads the occupied chunks of Phi (mostly from L2); "
                                       "writes the o tiles (0.49 GB) that oz_vgemm_kernel's epilogue reads",
                 "oz_vgemm_kernel": "reads: the o tiles (0.49 GB) plus the int8 slices re-read by tile CTAs, partly from L2; "
                                    "writes: the pair f values for the guard's refinement pass (67 MB) and the partials",
                 "oz_slice_kernel": "reads Phi (occupied and virtual rows); writes 7 int8 slices per row in the UMMA layout"}
        traffic = {"kernel": k, "config": "cfg4 (m=2048)", "dram_bytes_per_launch": int(r + w),
                   "dram_read_bytes": int(r), "dram_write_bytes": int(w),
                   "source": f"ncu --set full --clock-control none, gpurun_out/{rep.name}, one steady-state launch",
                   "note": notes.get(k, "")}
        (ROOT / "profiles" / f"traffic_cfg4_{TRAFFIC_NAME.get(k, k)}.json").write_text(json.dumps(traffic, indent=1) + "\n")
        details = subprocess.run(["ncu", "-i", str(rep), "--page", "details", "--csv"], capture_output=True, text=True,
                                 check=True).stdout
        (ROOT / "profiles" / f"{tag}_{k}_ncu_details.csv").write_text(details)
    (ROOT / "profiles" / f"{tag}_ncu_raw_summary_cfg4.txt").write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1])
