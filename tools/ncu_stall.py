import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern, "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
for i, r in enumerate(rows):
    if "Address" in r and "Source" in r:
        hdr = r; start = i + 1; break
stall_cols = [c for c in hdr if c.startswith("stall_") or "Stall" in c]
agg = {}
data = []
for r in rows[start:]:
    if len(r) != len(hdr) or "Address" in r: continue
    d = dict(zip(hdr, r))
    try: float(d["Warp Stall Sampling (All Samples)"] or 0)
    except ValueError: continue
    data.append(d)
# aggregate stall reasons across kernel
cols = [c for c in hdr if c not in ("Address", "Source") and c.startswith("Warp Stall Sampling") is False]
reason_cols = [c for c in hdr if "stall" in c.lower() and "Sampling" not in c]
tot = {}
for d in data:
    for c in reason_cols:
        try: tot[c] = tot.get(c, 0) + float(d[c] or 0)
        except ValueError: pass
for c, v in sorted(tot.items(), key=lambda x: -x[1])[:12]: print(f"{v:10.0f}  {c}")
