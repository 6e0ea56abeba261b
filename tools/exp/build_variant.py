"""Build an A/B variant of libpdm_b200.so with extra nvcc defines:
    python tools/exp/build_variant.py NAME -DFOO=1 ...
-> paper_2407_21552_b200/lib/variants/libpdm_b200_NAME.so (select it at run
time with PDM_LIB_PATH=...)."""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import __graft_entry__ as g  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out = g.PKG / "lib" / "variants" / f"libpdm_b200_{name}.so"
objd = ROOT / "build" / "variants" / name
objd.mkdir(parents=True, exist_ok=True)
out.parent.mkdir(parents=True, exist_ok=True)
srcs = sorted(g.CSRC.glob("*.cu")) + sorted(g.CSRC.glob("*.cpp"))


def one(src):
    obj = objd / (src.stem + ".o")
    cmd = [g._nvcc(), *g.NVCC_FLAGS, *g.FILE_FLAGS.get(src.name, []), *defs, "-c", str(src),
           "-o", str(obj)]
    subprocess.run(cmd, check=True)
    return obj


with ThreadPoolExecutor(8) as ex:
    objs = list(ex.map(one, srcs))
subprocess.run([g._nvcc(), "-shared", *g.NVCC_FLAGS[:2], "-o", str(out), *map(str, objs),
                "-lpthread"], check=True)
print(out)
