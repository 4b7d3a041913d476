"""Summarise an ncu --set full report into profiles/ncu_summary.json (read by
bench.py for roofline.traffic) and print the key metrics."""
import csv, json, subprocess, sys
rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
units = rows[1]
res = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    # "void oea_dev::k_ffn_bf16<2>(oea_dev::FfnParams)" -> "k_ffn_bf16<2>"
    key = name.split("(")[0].replace("void ", "").replace("oea_dev::", "").strip()
    d = {}
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if u == "Mbyte": v *= 1e6
            elif u == "Gbyte": v *= 1e9
            elif u == "Kbyte": v *= 1e3
            elif u == "usecond" or u == "us": v *= 1e3  # -> ns
            elif u == "msecond" or u == "ms": v *= 1e6
            d[w] = v
    res.setdefault(key, []).append(d)
summary = {}
for k, lst in res.items():
    avg = {m: sum(x.get(m, 0) for x in lst) / len(lst) for m in lst[0]}
    if "dram__bytes_read.sum" in avg:
        avg["dram_bytes_per_launch"] = avg["dram__bytes_read.sum"] + avg.get("dram__bytes_write.sum", 0)
    avg["launches_captured"] = len(lst)
    summary[k] = avg
summary["_source"] = "ncu --set full --clock-control none (tools/profile_decode.py, C1 shape, OEA simplified(4,8), cold-cache replay)"
json.dump(summary, open(out, "w"), indent=1)
for k, v in summary.items():
    if isinstance(v, dict):
        print(k, {m: (round(x, 3) if isinstance(x, float) else x) for m, x in v.items()})
