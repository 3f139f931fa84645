"""Per-launch DRAM traffic (usage: ncu_traffic.py REPORT [REPORT ...] OUT.json) (dram__bytes_read.sum + dram__bytes_write.sum) of the chain kernels from
one `ncu --set full` capture of tools/profile_step.py, keyed by the bench trace names ->
profiles/ncu_traffic.json (read by bench.py for roofline.traffic)."""
import csv
import json
import subprocess
import sys

reps, out = sys.argv[1:-1], sys.argv[-1]     # several reports merge (first capture of a name wins)
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
res = {}
for rep in reps:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    ik = hdr.index("Kernel Name")
    ir, iw, it = (hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum"),
                  hdr.index("gpu__time_duration.sum"))
    resid_seen = 0
    for r in rows[2:]:
        k = r[ik]
        if "gemm_bf16_tc<6" in k:
            name = "gemm_qkv"
        elif "gemm_bf16_tc<4" in k:
            name = "gemm_gate_up"
        elif "gemm_bf16_tc<1" in k:
            name = "gemm_o" if resid_seen == 0 else "gemm_down"
            resid_seen += 1
        elif "gemm_pair_tc<0" in k or "gemm_bf16_tc<0" in k:
            name = "gemm_head"
        elif "attn_paged" in k:
            name = "attention"
        elif "kv_relocate" in k:
            name = "kv_relocate"
        elif "rmsnorm" in k:
            name = "rmsnorm"
        else:
            continue
        if name in res:
            continue
        b = float(r[ir].replace(",", "")) * scale[units[ir]] + float(r[iw].replace(",", "")) * scale[units[iw]]
        res[name] = {"dram_bytes": int(b),
                     "ncu_duration_us": float(r[it].replace(",", "")) / (1e3 if units[it] == "nsecond" else 1),
                     "kernel": k.split("(")[0]}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
