"""Stall samples per CUDA source line from `ncu -i REP --page source --csv --print-source cuda,sass`:
    python tools/exp/ncu_lines.py SOURCE.csv [TOP]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
f = None; hdr = None; out = []
for r in rows:
    if not r: continue
    if r[0] == "File Path": f = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or r[0] == "" or r[0] == "Function Name": continue
    d = dict(zip(hdr[2:], r[2:]))  # note duplicated 'Source'
    try: s = int(d["Warp Stall Sampling (All Samples)"])
    except: continue
    st = {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit() and int(v) > 0}
    out.append((s, f, r[0], r[1][:90], st, d.get("Instructions Executed")))
tot = sum(o[0] for o in out)
print("total samples", tot)
for o in sorted(out, reverse=True)[:int(sys.argv[2]) if len(sys.argv)>2 else 40]:
    top = sorted(o[4].items(), key=lambda x: -x[1])[:4]
    print("%6d %5.1f%% %s:%s inst=%s | %s | %s" % (o[0], 100*o[0]/tot, o[1], o[2], o[5], o[3].strip(), " ".join("%s=%d"%(k[6:],v) for k,v in top)))
