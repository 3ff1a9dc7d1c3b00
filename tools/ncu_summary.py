"""Summarise ncu outputs into profiles/ (committed evidence).
    python tools/ncu_summary.py --launches gpurun_out/launches.csv --rep gpurun_out/prof.ncu-rep --tag r1_v0
Writes profiles/<tag>_launches.md (per-kernel share of device time, cold/serialised),
profiles/<tag>_ncu.md (key counters per profiled launch) and updates profiles/ncu_traffic.json
(per-launch dram bytes of k_push / k_select, used by bench.py's roofline.traffic)."""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_sectors_srcunit_tex_op_red.sum",
        "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed_op_global_red.sum", "smsp__inst_executed.sum",
        "lts__t_tag_requests.max.pct_of_peak_sustained_elapsed",
        "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        v = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
        agg[d["Kernel Name"].split("(")[0]][0] += 1
        agg[d["Kernel Name"].split("(")[0]][1] += v
    tot = sum(t for _, t in agg.values())
    lines = ["| kernel | launches | total ms | avg us | share |", "|---|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {c} | {t / 1e6:.3f} | {t / c / 1e3:.2f} | {t / tot:.3f} |")
    return "\n".join(lines)


def counters(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        e = {"kernel": d[hdr.index("Kernel Name")].split("(")[0]}
        for k in KEYS:
            if k in hdr:
                e[k] = d[hdr.index(k)] + (" " + units[hdr.index(k)] if units[hdr.index(k)] else "")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
                try:
                    stalls.append((float(d[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        e["top_stalls"] = [f"{n}:{int(v)}" for v, n in sorted(stalls, reverse=True)[:4]]
        res.append(e)
    return res


def to_bytes(s):
    v, u = s.split()[0], (s.split()[1] if len(s.split()) > 1 else "byte")
    return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--tag", required=True)
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    if a.launches:
        with open(os.path.join(ROOT, "profiles", f"{a.tag}_launches.md"), "w") as f:
            f.write(f"# {a.tag}: ncu launch list (gpu__time_duration.sum, --clock-control none; cold, serialised)\n\n")
            f.write(launches(a.launches) + "\n")
    if a.rep:
        c = counters(a.rep)
        with open(os.path.join(ROOT, "profiles", f"{a.tag}_ncu.md"), "w") as f:
            f.write(f"# {a.tag}: ncu --set full key counters per profiled launch\n\n")
            for e in c:
                f.write(f"## {e['kernel']}\n")
                for k, v in e.items():
                    if k != "kernel":
                        f.write(f"- {k}: {v}\n")
                f.write("\n")
        tr_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        try:
            old = json.load(open(tr_path))
        except Exception:
            old = {}
        tr = {}
        for e in c:
            name = e["kernel"].split("::")[-1].split("(")[0].strip()
            # the single-GPU plain instantiations keep the short key bench.py reads ("k_cycle":
            # k_cycle<0, 0, 0, 0> or r1's k_cycle<0, 0>, and round 2's warm-tier k_cycle<0, 0, 0, 0, 1>,
            # the bench kernel on C4); other instantiations (COLD, DIST, LOOPS) get their template
            # arguments in the key
            base, _, targs = name.partition("<")
            targs = targs.rstrip(">").replace(" ", "")
            plain = not targs or set(targs.split(",")) == {"0"} or targs == "0,0,0,0,1"
            name = base if plain else f"{base}<{targs}>"
            b = to_bytes(e["dram__bytes_read.sum"]) + to_bytes(e["dram__bytes_write.sum"])
            tr.setdefault(name + "_samples", []).append(b)
        for k in list(tr):
            if k.endswith("_samples"):
                tr[k[:-8]] = sum(tr[k]) / len(tr[k])  # mean over the captured launches
                old[k[:-8] + "_source"] = f"profiles/{a.tag}_ncu.md"
        old.update(tr)
        old.pop("source", None)
        json.dump(old, open(tr_path, "w"), indent=1)
    print("ok")
