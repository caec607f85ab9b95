"""SASS rows of an ncu source page exported with --print-source cuda,sass --csv:
address, warp-level executed count, avg active threads, stall samples, instruction,
owning source line.  Usage: sass_lines.py CSV [min_exec]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
mn = float(sys.argv[2]) if len(sys.argv) > 2 else 0
cur_file, cur_line, hdr, out = None, None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("Function Name", "Kernel Name"):
        continue
    if r[0].strip():
        cur_line = f"{cur_file}:{r[0]}"
        continue
    if len(r) > 8 and r[2].startswith("0x"):
        ex = float(r[7] or 0)
        th = float(r[8] or 0)
        out.append((int(r[2], 16), ex, th / ex if ex else 0, float(r[4] or 0), r[3].strip(), cur_line))
out.sort()
tot = sum(o[1] for o in out)
print(f"total warp instr {tot:.4e}")
base = out[0][0] if out else 0
for a, ex, avg, st, ins, ln in out:
    if ex >= mn:
        print(f"{a-base:6x} {ex:10.3e} {avg:5.1f} {st:6.0f}  {ins[:60]:60s} {ln}")
