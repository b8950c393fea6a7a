# Per-kernel SASS instruction summary of libinfllm_b200.so (cuobjdump -sass):
# counts of the Blackwell-native instructions (tcgen05 MMA / TMEM moves / TMA /
# bulk copies / mma.sync / fp64) and resource usage, as Markdown.
#   python tools/sass_summary.py > profiles/r02_sass_summary.md
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2402_04617_b200/libinfllm_b200.so"
KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "HMMA", "DFMA", "DADD",
        "MUFU.EX2", "FFMA2", "FADD2", "SHFL", "BAR.SYNC", "SYNCS"]
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
usage = {}
for m in re.finditer(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+) SHARED:(\d+)", res):
    usage[m.group(1)] = (int(m.group(2)), int(m.group(3)), int(m.group(4)))
funcs = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]+\*/\s+(@!?P\w+\s+)?([A-Z0-9_.]+)", line)
    if m:
        op = m.group(2)
        for k in KEYS:
            if op == k or op.startswith(k + "."):
                funcs[cur][k] += 1
        funcs[cur]["total"] += 1


def short(name):
    m = re.search(r"(k_\w+?)(E|I|P|$)", name)
    return m.group(1) if m else name[:40]


rows = [(short(f), f, c) for f, c in funcs.items() if short(f).startswith("k_")]
print("# SASS instruction summary, libinfllm_b200.so (sm_100a)\n")
print(f"`cuobjdump -sass {LIB}` per kernel: counts of static instructions (not executed counts).")
print("UTCHMMA = tcgen05.mma, LDTM/STTM = tcgen05.ld/st (TMEM), UTMALDG = TMA tensor load (.MULTICAST across")
print("the cluster), UBLKCP = cp.async.bulk, HMMA = mma.sync, MUFU.EX2 = exp2, FFMA2/FADD2 = packed fp32 pairs.\n")
print("| kernel | regs | stack | smem (static) | " + " | ".join(KEYS) + " | instructions |")
print("|---" * (len(KEYS) + 5) + "|")
for s, f, c in sorted(rows):
    u = usage.get(f, (0, 0, 0))
    print(f"| {s} | {u[0]} | {u[1]} | {u[2]} | " + " | ".join(str(c.get(k, 0)) for k in KEYS) + f" | {c['total']} |")
mc = sum(1 for line in sass.splitlines() if "UTMALDG" in line and "MULTICAST" in line)
print(f"\nUTMALDG with .MULTICAST (whole library): {mc}")
