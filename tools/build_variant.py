"""Diagnostic builds for A/B experiments (never the product): copies the
package to OUT_DIR/paper_1207_1571_b200 and compiles libfvb.so there with
extra -D flags.  Run a tool against it with FVB_PKG_ROOT=OUT_DIR.

    python tools/build_variant.py OUT_DIR -DFVB_DIAG_FENCE ...
"""
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(os.path.dirname(HERE), "paper_1207_1571_b200")
sys.path.insert(0, PKG)
import build  # noqa: E402

out, defs = sys.argv[1], sys.argv[2:]
dst = os.path.join(out, "paper_1207_1571_b200")
if os.path.exists(dst):
    shutil.rmtree(dst)
shutil.copytree(PKG, dst, ignore=shutil.ignore_patterns("*.so", "__pycache__"))
srcs = [os.path.join(PKG, "csrc", s) for s in build.SOURCES]
cmd = [build.NVCC, *build.FLAGS, *defs, "-o", os.path.join(dst, "libfvb.so"), *srcs]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.stderr.write(r.stdout + r.stderr)
    sys.exit(1)
print(dst)
