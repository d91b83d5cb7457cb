import os, subprocess, sys
def ok(a, b):
    r = subprocess.run([sys.executable, "tools/repro_c5slice.py", str(a), str(b)], capture_output=True,
                       text=True, env={**os.environ, "CUDA_LAUNCH_BLOCKING": "1"}, timeout=300)
    print("probe", a, b, r.returncode, r.stdout.strip()[-120:], flush=True)
    return r.returncode == 0
a, b = 0, 296
print("full", ok(a, b), flush=True)
# shrink from the right, then from the left
while b - a > 1:
    m = (a + b) // 2
    if not ok(a, m):
        b = m
    elif not ok(m, b):
        a = m
    else:
        print("needs a combination across", a, m, b, flush=True)
        break
print("final", a, b, flush=True)
