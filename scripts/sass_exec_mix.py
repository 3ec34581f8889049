"""Executed SASS instruction mix of one kernel in an ncu report (source page):
thread-instructions per opcode, and per 32-bit word when the word count is
given.  python scripts/sass_exec_mix.py report.ncu-rep [words]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
words = float(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
isrc, ith = hdr.index("Source"), hdr.index("Predicated-On Thread Instructions Executed")
mix = collections.Counter()
for r in rows[2:]:
    if len(r) <= ith or not r[ith].strip().isdigit():
        continue
    op = r[isrc].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    mix[o.split(".")[0]] += int(r[ith])
tot = sum(mix.values())
for o, c in mix.most_common(16):
    print(f"{o:10s} {c:18d} {c / tot:6.1%}" + (f"  {c / words:8.3f} per word" if words else ""))
print(f"{'total':10s} {tot:18d}" + (f"        {tot / words:8.3f} per word" if words else ""))
