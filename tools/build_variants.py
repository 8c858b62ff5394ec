"""Build path-kernel variants for A/B timing.

    python tools/build_variants.py [N ...]             libmcsbr_gpu_v<N>.so (MCSBR_MIN_BLOCKS=N)
    python tools/build_variants.py --stats             libmcsbr_gpu_stats.so (traversal counters)
    python tools/build_variants.py --name X -DA=1 ...  libmcsbr_gpu_X.so with extra defines
    python tools/build_variants.py --name X --src DIR  sources in DIR override csrc/ (A/B vs an
                                                       older revision: git show REV:... > DIR/)
Time one with MCSBR_GPU_LIB=<so> python tools/profile_c2.py."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2511_07586_b200 import build as B  # noqa: E402

stats = "--stats" in sys.argv
name = sys.argv[sys.argv.index("--name") + 1] if "--name" in sys.argv else None
src_dir = sys.argv[sys.argv.index("--src") + 1] if "--src" in sys.argv else None
defines = [a for a in sys.argv[1:] if a.startswith("-D")]
args = [a for a in sys.argv[1:] if not a.startswith("-") and a not in (name, src_dir)]
for mb in [int(x) for x in args] or ([4] if name else [1, 2, 3, 4]):
    objs = []
    extra = (["-DMCSBR_TRAVERSAL_STATS"] if stats else []) + defines
    for src in B.SOURCES:
        obj = f"/tmp/v{mb}_{name or ("stats" if stats else "mb")}_{src}.o"
        path = os.path.join(B.CSRC, src)
        inc = []
        if src_dir:
            inc = ["-I", src_dir]
            if os.path.exists(os.path.join(src_dir, src)):
                path = os.path.join(src_dir, src)
        r = subprocess.run([B.NVCC, *inc, *B.FLAGS, *extra, f"-DMCSBR_MIN_BLOCKS={mb}", "-c",
                            path, "-o", obj], capture_output=True, text=True)
        if r.returncode:
            sys.exit(r.stderr[-3000:])
        if src == "trace.cu":
            print(mb, [l.strip() for l in r.stderr.splitlines() if "registers" in l][-3:])
        objs.append(obj)
    out = os.path.join(B.HERE, f"libmcsbr_gpu_{name}.so" if name else
                       "libmcsbr_gpu_stats.so" if stats else f"libmcsbr_gpu_v{mb}.so")
    subprocess.run([B.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs,
                    "-Xcompiler", "-fPIC", "-Xlinker", "--exclude-libs,ALL", "-Xlinker", "-Bsymbolic",
                    "-lcudart_static", "-lrt", "-lpthread", "-ldl"], check=True)
