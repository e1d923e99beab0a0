"""Aggregate ncu source-page samples per CUDA source line (cuda,sass view)."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import csv, subprocess, sys, collections
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source=cuda,sass'],
                     capture_output=True, text=True).stdout
cur_file, cur_line, cur_src = None, None, None
samp = collections.Counter(); execd = collections.Counter(); srcs = {}
hdr = None
for row in csv.reader(txt.splitlines()):
    if not row:
        continue
    if row[0] == 'File Path':
        cur_file = row[1].split('/')[-1]; continue
    if row[0] in ('Function Name',):
        continue
    if row[0] == 'Line No':
        hdr = row; continue
    if hdr is None:
        continue
    if row[0]:
        cur_line = int(row[0]); cur_src = row[1]
        srcs[(cur_file, cur_line)] = cur_src
        continue
    d = dict(zip(range(len(row)), row))
    try:
        s = int(row[hdr.index('# Samples')]); e = int(row[hdr.index('Instructions Executed')])
    except Exception:
        continue
    samp[(cur_file, cur_line)] += s; execd[(cur_file, cur_line)] += e
tot = sum(samp.values()); te = sum(execd.values())
print(f"total samples {tot}  warp-instructions {te}")
for k, v in samp.most_common(top):
    print(f"{100*v/tot:5.1f}% samp {100*execd[k]/max(te,1):5.1f}% inst  {k[0]}:{k[1]:4d}  {srcs.get(k,'')[:90]}")
