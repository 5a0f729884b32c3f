"""Build variants of one CUDA source with extra -D flags, each linked with the library's other
objects into build/variants/<name>/libflowtree_b200.so (select with FT_LIB=... at run time).
python tools/variants.py ft_flowd.cu name1:-DX=1,-DY=2 name2:-DX=3"""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_04126_b200 import build as B  # noqa: E402

B.build()
src = os.path.join(B.CSRC, sys.argv[1])
objs = [os.path.join(B.OBJ, os.path.basename(f)[:-3] + ".o") for f in B._sources()]
for spec in sys.argv[2:]:
    name, _, flags = spec.partition(":")
    d = os.path.join(B.ROOT, "build", "variants", name)
    os.makedirs(d, exist_ok=True)
    obj = os.path.join(d, os.path.basename(src)[:-3] + ".o")
    cmd = [B.NVCC] + B.ARCH + B.FLAGS + [f for f in flags.split(",") if f] + ["-c", src, "-o", obj]
    p = subprocess.run(cmd, capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    regs = [l for l in p.stderr.splitlines() if "registers" in l]
    lo = [obj if os.path.basename(o) == os.path.basename(obj) else o for o in objs]
    subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", os.path.join(d, "libflowtree_b200.so")] + lo, check=True)
    print(name, flags, regs[-1].strip() if regs else "")
