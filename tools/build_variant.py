"""Build an experiment variant of the native library with extra nvcc flags:

    python tools/build_variant.py NAME -DFLAG=1 ...  ->  paper_2501_08582_b200/_native/exp/NAME/liblors_b200.so

Run it with LORS_B200_LIB=<that path> (paper_2501_08582_b200/_native.py) to A/B against the default build."""
import concurrent.futures as cf
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_08582_b200 import build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
out = os.path.join(B.OUT_DIR, "exp", name)
os.makedirs(out, exist_ok=True)
objs = [os.path.join(out, s.replace(".cu", ".o")) for s in B.SOURCES]
cmds = [[B.nvcc(), *B.NVCC_FLAGS, *flags, "-c", os.path.join(B.CSRC, s), "-o", o] for s, o in zip(B.SOURCES, objs)]
with cf.ThreadPoolExecutor(len(cmds)) as ex:
    for r in ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds):
        if r.returncode:
            sys.exit(r.stderr)
subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", os.path.join(out, "liblors_b200.so"), *objs], check=True)
print(os.path.join(out, "liblors_b200.so"))
