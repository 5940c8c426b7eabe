"""Summarise ptxas -v logs: registers, stack frame and spills per kernel."""
import re, subprocess, sys, glob

def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.splitlines()

rows = []
for log in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "build/obj/*.ptxas.log")):
    cur = None
    for line in open(log):
        m = re.search(r"Function properties for (\S+)", line)
        if m: cur = m.group(1); continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur: rows.append([cur, *map(int, m.groups()), 0]); continue
        m = re.search(r"Used (\d+) registers", line)
        if m and rows and rows[-1][0] == cur: rows[-1][4] = int(m.group(1))
names = demangle([r[0] for r in rows])
only_bad = "--all" not in sys.argv
for n, r in zip(names, rows):
    if only_bad and r[1] == 0 and r[2] == 0: continue
    print(f"{r[4]:4d} regs stack {r[1]:5d} spillS {r[2]:5d} spillL {r[3]:5d}  {n[:110]}")
