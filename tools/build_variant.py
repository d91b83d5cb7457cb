"""Build a compile-time variant of the C-ABI library for an A/B run.

    python tools/build_variant.py <tag> -DNAME=VALUE ...
    SMG_LIB=paper_2402_12947_b200/lib/libsimplexmg_b200_<tag>.so python bench.py ...

The product build (build_lib.py) is untouched; variants live beside it in
lib/ (git-ignored, travels to the GPU box with the snapshot).
"""

import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_12947_b200 import build_lib  # noqa: E402


def main():
    tag, defines = sys.argv[1], sys.argv[2:]
    out = os.path.join(build_lib.LIBDIR, f"libsimplexmg_b200_{tag}.so")
    res = subprocess.run([build_lib.NVCC] + build_lib.COMPILE_FLAGS + build_lib.LINK_FLAGS[2:] + defines + ["-o", out]
                         + build_lib.sources(), capture_output=True, text=True)
    if res.returncode:
        sys.exit(res.stderr[-4000:])
    with open(out + ".ptxas.log", "w") as f:
        f.write(res.stderr)
    print(out)


if __name__ == "__main__":
    main()
