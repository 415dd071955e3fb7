"""Summarise ncu outputs into profiles/: launch-list shares per kernel and key
metrics of --set full captures (read here, no GPU needed)."""
import collections, csv, io, json, subprocess, sys

def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = collections.Counter(); cnt = collections.Counter()
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].split("<")[0].replace("void ", "").strip()
        if "k_attn<" in r[ki]:
            name = "k_attn<" + r[ki].split("k_attn<")[1].split(">")[0] + ">"
        if "k_attn_fusion_pair" in r[ki]:
            name = "k_attn_fusion_pair"
        elif "k_attn_pers<" in r[ki]:
            args = r[ki].split("k_attn_pers<")[1].split(">")[0].replace("(int)", "").split(",")
            name = "k_attn_pers<d_h=%s, %s>" % (args[0].strip(), "SUMI" if args[1].strip() == "0" else "HIST")
        elif "k_attn_fa<" in r[ki]:
            args = r[ki].split("k_attn_fa<")[1].split(">")[0].replace("(int)", "").split(",")
            name = "k_attn_fa<d_h=%s, %s>" % (args[0].strip(), "SUMI" if args[1].strip() == "0" else "HIST")
        if "k_gemm_tc<" in r[ki]:
            name = "k_gemm_tc<" + r[ki].split("k_gemm_tc<")[1].split(">")[0] + ">"
        v = float(r[vi].replace(",", ""))
        unit = hdr  # ns by default in ncu csv for duration
        tot[name] += v; cnt[name] += 1
    s = sum(tot.values())
    return {k: {"launches": cnt[k], "total": tot[k], "share": tot[k] / s} for k, _ in tot.most_common()}

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "smsp__inst_executed_pipe_xu", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform", "sm__pipe_shared_cycles_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"]

def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for h, u, v in zip(hdr, units, r):
            if any(h.startswith(k) for k in KEYS):
                d[h] = f"{v} {u}".strip()
        res.append(d)
    return res

if __name__ == "__main__":
    res = {"launch_shares": launches(sys.argv[1])}
    for p in sys.argv[2:]:
        res[p.split("/")[-1]] = full(p)
    print(json.dumps(res, indent=1))
