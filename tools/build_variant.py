"""Build kernel variants of one source file for A/B timing on the GPU box.

    python tools/build_variant.py region "-DUT_IM_SLEEP=1000" v1 ["-D..." v2 ...]

Each variant recompiles csrc/<src>.cu with the extra flags and links it with the
other objects of the normal build into scratch/lib_<name>.so; select one at run
time with UT_LIB_PATH=scratch/lib_<name>.so.
"""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_1612_06457_b200 import build as b  # noqa: E402

b.build()
src = sys.argv[1]
pairs = list(zip(sys.argv[2::2], sys.argv[3::2]))
out = ROOT / "scratch"
out.mkdir(exist_ok=True)
nvcc = b.nvcc_path()


def one(pair):
    flags, name = pair
    obj = out / f"{src}_{name}.o"
    cmd = [nvcc, *b.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I",
           str(b.INCLUDE), "--expt-relaxed-constexpr", *flags.split(), "-c",
           str(b.CSRC / f"{src}.cu"), "-o", str(obj)]
    subprocess.run(cmd, check=True)
    objs = [str(obj)] + [str(p) for p in sorted(b.OBJ_DIR.glob("*.o")) if p.stem != src]
    subprocess.run([nvcc, *b.ARCH, "-shared", "-cudart", "static", "-o",
                    str(out / f"lib_{name}.so"), *objs], check=True)
    return name


with ThreadPoolExecutor(max_workers=4) as pool:
    for n in pool.map(one, pairs):
        print("built", n)
