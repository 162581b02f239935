"""Summarise an ncu --set full report: per kernel duration, DRAM bytes,
throughputs, occupancy.  Writes a markdown table and the traffic json."""
import csv, io, json, subprocess, sys
rep, out_md, out_json = sys.argv[1], sys.argv[2], sys.argv[3]
CFG = sys.argv[4] if len(sys.argv) > 4 else "C3"
# kernel (name prefix in the report) -> bench.py `kernels` key; first launch of each
KEYS = [("k_span<2, 0, 1", "fine_spmv"), ("k_span<2, 2, 0", "fine_presmooth"), ("k_csr<1, 2, 4", "fine_prolongation"),
        ("k_span<2, 3, 1", "fine_postsmooth"), ("k_csr<4, 2, 0", "fine_restriction"),
        ("k_csr<4, 2, 1", "level1_presmooth"), ("k_csr<4, 2, 6", "level1_prolong_post"),
        ("k_update_r<2>", "pcg_r_update"), ("k_xpby_x<2>", "pcg_p_update")]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
cols = {k: h.index(k) for k in ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                  "l1tex__throughput.avg.pct_of_peak_sustained_active",
                                  "lts__throughput.avg.pct_of_peak_sustained_elapsed",
                                  "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
                                  "launch__grid_size"]}
units = rows[1]
def val(r, k):
    v = float(r[cols[k]].replace(",", ""))
    u = units[cols[k]]
    if u == "Mbyte": v *= 1e6
    elif u == "Gbyte": v *= 1e9
    elif u == "Kbyte": v *= 1e3
    elif u == "ms": v *= 1e3
    elif u == "ns": v /= 1e3
    return v
lines = ["| kernel | us | DRAM read MB | DRAM write MB | DRAM GB/s | L1 % | L2 % | warps active % | regs | grid |",
         "|---|---|---|---|---|---|---|---|---|---|"]
traffic = {}
for r in rows[2:]:
    name = r[cols["Kernel Name"]].split("(")[0].replace("void ", "").replace("unnamed>::", "")
    us = val(r, "gpu__time_duration.sum")
    rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
    lines.append(f"| `{name}` | {us:.1f} | {rd/1e6:.1f} | {wr/1e6:.1f} | {(rd+wr)/us/1e3:.0f} | "
                 f"{float(r[cols['l1tex__throughput.avg.pct_of_peak_sustained_active']]):.0f} | "
                 f"{float(r[cols['lts__throughput.avg.pct_of_peak_sustained_elapsed']]):.0f} | "
                 f"{float(r[cols['sm__warps_active.avg.pct_of_peak_sustained_active']]):.0f} | "
                 f"{r[cols['launch__registers_per_thread']]} | {r[cols['launch__grid_size']]} |")
    for prefix, key in KEYS:
        if name.startswith(prefix) and f"{CFG}_{key}_dram_bytes" not in traffic:
            traffic[f"{CFG}_{key}_dram_bytes"] = rd + wr
            traffic[f"{CFG}_{key}_ncu_us"] = us
open(out_md, "w").write("\n".join(lines) + "\n")
json.dump(traffic, open(out_json, "w"), indent=1)
print("\n".join(lines)); print(traffic)
