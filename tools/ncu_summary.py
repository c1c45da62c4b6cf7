"""Summarise an ncu report (`--set full`) for profiles/: per kernel the
duration, DRAM bytes read/written, DRAM and tensor-pipe utilisation, SM
throughput, occupancy and registers.  Emits text and a JSON record.

    python tools/ncu_summary.py report.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pct_rt",
    "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg": "tensor_hmma_cycles",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_mem_pct",
    "sm__cycles_elapsed.avg": "cycles_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "tc_smem_pct",
    "sm__inst_executed_pipe_tensor_op_hmma.avg.pct_of_peak_sustained_active": "hmma_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_lsu_pct",
    "smsp__inst_executed.sum": "inst_executed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pct",
}


def main(path, json_out=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        rec = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for i, h in enumerate(hdr):
            h = h.split(".", 2)[-1] if h.startswith(("TPC.", "SM_C.", "GPC.")) else h
            if h in WANT:
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if h.startswith("dram__bytes"):
                    v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                if h == "gpu__time_duration.sum":
                    v *= {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(u, 1)
                rec[WANT[h]] = v
        recs.append(rec)
    for rec in recs:
        print(rec["kernel"])
        for k, v in rec.items():
            if k != "kernel":
                print(f"    {k:22s} {v:,.3f}" + (" us" if k == "duration" else ""))
        if "dram_read" in rec and "dram_write" in rec:
            print(f"    {'dram_bytes_total':22s} {rec['dram_read'] + rec['dram_write']:,.0f}")
    if json_out:
        with open(json_out, "w") as fh:
            json.dump(recs, fh, indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[3] if len(sys.argv) > 3 and sys.argv[2] == "--json" else None)
