"""Per-kernel SASS opcode counts of the built library (static instruction
counts, not executed): DMMA (FP64 tensor pipe), DFMA/DADD/DMUL (FP64 CUDA
cores), UTMALDG/UBLKCP/UBLKPF (TMA copy / bulk L2 prefetch), CREDUX (warp reductions), LDGSTS (cp.async), LDS/STS, BAR, SHFL.

    python tools/sass_counts.py [lib.so] > profiles/rNN_sass_counts.txt
"""
import collections, os, re, subprocess, sys  # noqa: E401

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1110_3105_b200", "libskel_sm100.so")
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
OPS = ["DMMA", "DFMA", "DADD", "DMUL", "UTMALDG", "UBLKCP", "UBLKPF", "CREDUX", "SYNCS", "LDGSTS", "LDG", "STG", "LDS", "STS",
       "BAR", "SHFL", "MUFU"]
cur, counts = None, collections.OrderedDict()
for line in txt.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[\w.]+)?", line)
    if m:
        op = m.group(1)
        for k in OPS:
            if op == k:
                counts[cur][k] += 1
        counts[cur]["total"] += 1


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.splitlines()


names = list(counts)
pretty = demangle(names)
print("static SASS opcode counts per kernel (cuobjdump -sass " + os.path.basename(lib) + ")")
print("kernel | " + " ".join(OPS) + " total")
for raw, nice in sorted(zip(names, pretty), key=lambda t: t[1]):
    c = counts[raw]
    nice = re.sub(r"\(.*", "", nice)
    print(f"{nice[:90]} | " + " ".join(str(c[k]) for k in OPS) + f" {c['total']}")
