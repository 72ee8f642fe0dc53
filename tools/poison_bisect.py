"""dev: bisect the allocation index whose initial content changes a solve (poison 0 vs none)."""
import os, subprocess, sys
def run(lo, hi, poison=True):
    e = dict(os.environ)
    if poison:
        e.update(PINS_POISON="0", PINS_POISON_LO=str(lo), PINS_POISON_HI=str(hi))
    out = subprocess.run([sys.executable, "tools/initcheck_sparse.py", "2", "1"], env=e, capture_output=True, text=True)
    line = [l for l in out.stdout.splitlines() if l.startswith("obj")]
    return line[-1] if line else out.stderr[-300:]
base = run(0, 0, poison=False)
full = run(0, 1 << 40)
print("base", base, "| full poison", full, flush=True)
e = dict(os.environ); e.update(PINS_POISON_LIST="1")
out = subprocess.run([sys.executable, "tools/initcheck_sparse.py", "2", "1"], env=e, capture_output=True, text=True)
allocs = [l for l in out.stderr.splitlines() if l.startswith("alloc")]
print("allocations", len(allocs), flush=True)
lo, hi = 0, len(allocs)
while hi - lo > 1:
    mid = (lo + hi) // 2
    r = run(lo, mid)
    print(lo, mid, r, flush=True)
    if r != base: hi = mid
    else: lo = mid
print("culprit allocation", lo, allocs[lo] if lo < len(allocs) else None)
print("\n".join(allocs[max(0, lo - 3):lo + 4]))
