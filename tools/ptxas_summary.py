"""Summarise nvcc -Xptxas -v output: kernel, registers, spill bytes (stdin)."""
import re, subprocess, sys
cur = None
out = []
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = (int(m.group(1)), int(m.group(2)))
        out.append([cur, None, spill])
    m = re.search(r"Used (\d+) registers", line)
    if m and out and out[-1][1] is None:
        out[-1][1] = int(m.group(1))
for name, regs, spill in out:
    try:
        dn = subprocess.run(["c++filt"], input=name, capture_output=True, text=True).stdout.strip()
    except OSError:
        dn = name
    dn = re.sub(r"evr::MarchRows<.*", "", dn)
    print(f"{regs!s:>4} regs  spill st/ld {spill[0]:>4}/{spill[1]:<5} {dn[:110]}")
