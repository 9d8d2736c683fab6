"""Summarise `nvcc -Xptxas -v` output: registers / spills per kernel (stdin)."""
import re, sys
cur = None; spill = {}
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m: cur = m.group(1); continue
    m = re.search(r"Function properties for (\S+)", line)
    if m: cur = m.group(1); continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur: spill[cur] = (int(m.group(1)), int(m.group(2))); continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        name = cur
        try:
            import subprocess
            name = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        except Exception:
            pass
        name = re.sub(r"nsm::\(anonymous namespace\)::", "", name)
        print(f"{m.group(1):>4} regs  spill {spill.get(cur, (0, 0))}  {name[:110]}")
