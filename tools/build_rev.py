"""Build libhfmm_NAME.so from the library sources of git revision REV (A/B against older kernels):
    python tools/build_rev.py NAME REV    -> paper_0911_4114_b200/libhfmm_NAME.so"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_0911_4114_b200.build as B  # noqa: E402

name, rev = sys.argv[1], sys.argv[2]
tmp = tempfile.mkdtemp(prefix="hfmm_rev_")
os.makedirs(os.path.join(tmp, "pkg", "csrc"))   # same depth as the repo: csrc/../../include
os.makedirs(os.path.join(tmp, "include"))
for src in B.SOURCES + ["hfmm_impl.h"]:
    data = subprocess.check_output(["git", "-C", ROOT, "show", f"{rev}:paper_0911_4114_b200/csrc/{src}"])
    open(os.path.join(tmp, "pkg", "csrc", src), "wb").write(data)
open(os.path.join(tmp, "include", "hfmm.h"), "wb").write(
    subprocess.check_output(["git", "-C", ROOT, "show", f"{rev}:include/hfmm.h"]))
B.CSRC = os.path.join(tmp, "pkg", "csrc")
B.ROOT = tmp
out = os.path.join(B.HERE, f"libhfmm_{name}.so")
B.build(force=True, verbose=False, out=out)
print(out)
