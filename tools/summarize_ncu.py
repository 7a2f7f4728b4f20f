"""Summaries for profiles/: launch-list shares and per-kernel DRAM traffic.

usage: python tools/summarize_ncu.py launches <launches.csv> <command> > out.json
       python tools/summarize_ncu.py full <report.ncu-rep> <command> <pairs_per_launch> > out.json
"""
import collections, csv, io, json, subprocess, sys


def launches(path, command):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0}[d["Metric Unit"]]
                name = d["Kernel Name"].split("(")[0].replace("void <unnamed>::", "").replace("<unnamed>::", "")
                agg[name].append(float(d["Metric Value"]) * scale)
    tot = sum(sum(v) for v in agg.values())
    ks = [{"kernel": k, "launches": len(v), "ms": sum(v), "share": sum(v) / tot, "avg_ms": sum(v) / len(v)}
          for k, v in sorted(agg.items(), key=lambda t: -sum(t[1]))]
    return {"command": command, "ncu": "--metrics gpu__time_duration.sum --clock-control none "
            "(cold-cache, serialised launches: compare shares, not absolute times)",
            "total_ms": tot, "kernels": ks}


def full(path, command, pairs):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u = r[0], r[1]
    keys = {"gpu__time_duration.sum": "duration", "dram__bytes_read.sum": "dram_read",
            "dram__bytes_write.sum": "dram_write", "smsp__inst_executed.sum": "warp_instructions",
            "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
            "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
            "launch__registers_per_thread": "regs", "launch__grid_size": "grid"}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
    res = []
    for v in r[2:]:
        d = {}
        for k, name in keys.items():
            i = h.index(k)
            val = float(v[i].replace(",", ""))
            if u[i] in scale:
                val *= scale[u[i]]
            d[name + ("_ms" if name == "duration" else "_bytes" if name.startswith("dram") else "")] = val
        d["kernel"] = v[h.index("Kernel Name")].split("(")[0].replace("void <unnamed>::", "")
        d["pairs_per_launch"] = pairs
        d["dram_bytes_per_pair"] = (d["dram_read_bytes"] + d["dram_write_bytes"]) / pairs
        d["warp_instructions_per_pair"] = d["warp_instructions"] / pairs
        res.append(d)
    return {"command": command, "ncu": "--set full --clock-control none --import-source on", "launches": res}


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(json.dumps(launches(sys.argv[2], sys.argv[3]), indent=1))
    else:
        print(json.dumps(full(sys.argv[2], sys.argv[3], float(sys.argv[4])), indent=1))
