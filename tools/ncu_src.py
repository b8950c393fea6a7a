import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern, "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
for i, r in enumerate(rows):
    if "Address" in r and "Source" in r:
        hdr = r; start = i + 1; break
data = []
for r in rows[start:]:
    if len(r) != len(hdr) or "Address" in r:
        continue
    d = dict(zip(hdr, r))
    try:
        float(d["Warp Stall Sampling (All Samples)"] or 0)
    except ValueError:
        continue
    data.append(d)
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(d[key] or 0) for d in data) or 1
top = sorted(data, key=lambda d: -float(d[key] or 0))[:int(sys.argv[3]) if len(sys.argv) > 3 else 25]
for d in top:
    print(f"{float(d[key])/tot*100:5.1f}%  {d['Source'][:120]}")
