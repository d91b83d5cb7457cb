"""Bisect which patch sizes make apply_local_correction fail (each probe in a fresh process)."""
import subprocess, sys
def probe(sizes):
    arg = ",".join(map(str, sizes + [512]))
    r = subprocess.run([sys.executable, "tools/repro_lc.py", arg], capture_output=True, text=True,
                       env={**__import__("os").environ, "CUDA_LAUNCH_BLOCKING": "1"}, timeout=300)
    return r.returncode == 0 and "rel" in r.stdout
sizes = list(range(64, 513))
print("all sizes ok:", probe(sizes), flush=True)
lo = sizes
while len(lo) > 1:
    half = lo[:len(lo) // 2]
    rest = lo[len(lo) // 2:]
    if not probe(half):
        lo = half
    elif not probe(rest):
        lo = rest
    else:
        print("both halves pass separately; failing needs a combination:", lo[0], lo[-1], flush=True)
        break
    print("narrowed to", lo[0], "..", lo[-1], len(lo), flush=True)
print("result", lo[:10], flush=True)
