"""Build libcutfem_mg.so in-tree with nvcc for sm_100a (no JIT, no torch)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "capi.cu")
OUT = os.path.join(HERE, "libcutfem_mg.so")
DEPS = [os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))] + \
       [os.path.join(ROOT, "include", "cutfem_mg.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr",
         "-cudart", "shared"]


def needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force=False, verbose=False, out=None, extra=()):
    """Compile capi.cu into `out` (default: the in-tree library); `extra` =
    additional nvcc flags (e.g. -D variants for A/B timing runs)."""
    out = out or OUT
    if out == OUT and not force and not needs_build():
        return OUT
    cmd = [NVCC] + FLAGS + list(extra) + ["-I", os.path.join(ROOT, "include"), SRC, "-o", out + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = r.stdout + r.stderr
    with open(os.path.join(HERE, "build.log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + log)
    if r.returncode != 0:
        sys.stderr.write(log[-8000:])
        raise RuntimeError("nvcc failed (see paper_2508_11608_b200/build.log)")
    os.replace(out + ".tmp", out)
    if verbose:
        print(log)
    return out


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if a not in ("--force", "-v")]
    out = None
    if "--out" in args:
        i = args.index("--out")
        out = args[i + 1]
        del args[i:i + 2]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=out, extra=args))
