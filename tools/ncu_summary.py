"""Summarize ncu outputs into profiles/ (run in the build container).

  python tools/ncu_summary.py rep  <file.ncu-rep> <out.json>   # --set full capture
  python tools/ncu_summary.py list <launches.csv> <out.json>   # launch list
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
        "l1tex__t_bytes.sum", "lts__t_sectors_srcunit_tex_op_read.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1, "us": 1e3, "ms": 1e6}


def rep(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                v = r[i].replace(",", "")
                try:
                    val = float(v) * SCALE.get(units[i], 1)
                except ValueError:
                    val = v
                d[k + (" [ns]" if units[i] in ("ns", "us", "ms") else " [B]" if "byte" in units[i] else "")] = val
        launches.append(d)
    dram = [l["dram__bytes_read.sum [B]"] + l["dram__bytes_write.sum [B]"] for l in launches
            if "dram__bytes_read.sum [B]" in l]
    summary = {"source": path, "launches": launches,
               "dram_bytes_per_launch": sum(dram) / len(dram) if dram else None}
    json.dump(summary, open(out, "w"), indent=1)
    print(json.dumps(summary, indent=1)[:2000])


def launch_list(path, out):
    text = open(path).read()
    rows = list(csv.DictReader(io.StringIO(text[text.index('"ID"'):])))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = SCALE.get(r["Metric Unit"], 1)
        agg[r["Kernel Name"]][0] += 1
        agg[r["Kernel Name"]][1] += float(r["Metric Value"].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values())
    res = [{"kernel": k, "launches": n, "total_ns": t, "mean_ns": t / n, "share": t / tot}
           for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])]
    json.dump({"source": path, "kernels": res}, open(out, "w"), indent=1)
    for r in res:
        print(f"{r['launches']:5d} {r['mean_ns']/1e3:9.2f} us {100*r['share']:5.1f}%  {r['kernel'][:90]}")


if __name__ == "__main__":
    {"rep": rep, "list": launch_list}[sys.argv[1]](sys.argv[2], sys.argv[3])
