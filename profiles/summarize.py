"""Summarise ncu captures into the committed profile files.

  python profiles/summarize.py <prof.ncu-rep> <out_prefix> [launches.csv]

Writes <out_prefix>.md (human-readable key metrics per kernel) and merges the
search kernels' instruction counts into profiles/search_issue.json (read by
bench.py for the live ALU-issue roofline) and the texture kernel's DRAM bytes
into profiles/texture_traffic.json.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
KEYS = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Executed Instructions",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "L1/TEX Hit Rate", "L2 Hit Rate", "DRAM Throughput", "Memory Throughput",
        "No Eligible", "Warp Cycles Per Issued Instruction", "SM Frequency", "DRAM Frequency"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ki, sec, name, unit, val = (hdr.index("Kernel Name"), hdr.index("Section Name"),
                                hdr.index("Metric Name"), hdr.index("Metric Unit"),
                                hdr.index("Metric Value"))
    idi = hdr.index("ID")
    kern = {}
    for r in rows[1:]:
        if len(r) <= val:
            continue
        k = (r[idi], r[ki])
        kern.setdefault(k, {})[r[name]] = (r[val], r[unit], r[sec])
    return kern


def raw_metric(rep, metric):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", metric],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    mi = hdr.index(metric)
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(rows[1][mi], 1.0)
    res = []
    for r in rows[2:]:
        if len(r) > mi:
            res.append((r[hdr.index("Kernel Name")], float(r[mi].replace(",", "")) * scale))
    return res


def main():
    rep, prefix = sys.argv[1], sys.argv[2]
    kern = details(rep)
    lines = [f"# ncu summary: {os.path.basename(rep)}", ""]
    issue = {}
    for (kid, kname), m in kern.items():
        lines.append(f"## [{kid}] {kname}")
        for k in KEYS:
            if k in m:
                v, u, _ = m[k]
                lines.append(f"- {k}: {v} {u}")
        lines.append("")
        if "k_search" in kname or "k_trace_walk" in kname:
            if "k_trace_walk" in kname:  # the trace interpreters: walk = step 1, walk2 = step 2
                step = "2" if "k_trace_walk2" in kname else "1"
            else:
                mt = re.search(r"k_search<[^,]*,\s*(?:\(int\))?(\d)", kname)
                step = mt.group(1) if mt else "1"
            try:
                issue[f"warp_inst_step{step}"] = float(m["Executed Instructions"][0].replace(",", ""))
                issue[f"issue_active_pct_step{step}"] = float(m["Issue Slots Busy"][0])
                f, u = m.get("SM Frequency", ("0", "Mhz"))[:2]
                issue["sm_mhz_ncu"] = float(f) * (1000.0 if u.lower() == "ghz" else 1.0)
            except (KeyError, ValueError):
                pass
    try:
        rd = raw_metric(rep, "dram__bytes_read.sum")
        wr = raw_metric(rep, "dram__bytes_write.sum")
        lines.append("## DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)")
        for (k, a), (_, b) in zip(rd, wr):
            lines.append(f"- {k[:60]}: read {a:.0f} B, write {b:.0f} B")
            if "k_texture" in k:
                tj = os.path.join(HERE, "texture_traffic.json")
                d = json.load(open(tj)) if os.path.exists(tj) else {}
                d[os.environ.get("CFG", "cfg3")] = a + b
                json.dump(d, open(tj, "w"), indent=1)
            if "k_search" in k or "k_trace_walk" in k:
                issue.setdefault("dram_bytes_per_launch", a + b)
    except Exception as e:  # raw page layout differs across ncu versions
        lines.append(f"(raw dram metrics unavailable: {e})")
    open(prefix + ".md", "w").write("\n".join(lines) + "\n")
    if issue:
        sj = os.path.join(HERE, "search_issue.json")
        d = json.load(open(sj)) if os.path.exists(sj) else {}
        key = os.environ.get("KEY", "cfg3_mode0")
        if "issue_active_pct_step1" in issue:
            issue["issue_active_pct"] = issue["issue_active_pct_step1"]
        sys.path.insert(0, os.path.dirname(HERE))
        from bench import kernel_src_sha
        d[key] = {**d.get(key, {}), **issue, "source": os.path.basename(rep),
                  "kernel_src_sha": kernel_src_sha()}
        json.dump(d, open(sj, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
