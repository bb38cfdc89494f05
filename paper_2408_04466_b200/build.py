"""Build libgwn_b200.so in-tree with nvcc for sm_100a (no JIT cache)."""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libgwn_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    "-Xptxas", "-v",
    "-shared", "--expt-relaxed-constexpr",
]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(HERE, "csrc", "*.h")) + \
        glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + \
        [os.path.join(REPO, "include", "gwn_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(out: str, defines: list[str]) -> str:
    """Each .cu to an object in parallel (one nvcc per file), then one link."""
    from concurrent.futures import ThreadPoolExecutor
    odir = out + ".objs"
    os.makedirs(odir, exist_ok=True)
    base = [NVCC, *[f for f in FLAGS if f != "-shared"], *[f"-D{d}" for d in defines],
            "-I", os.path.join(REPO, "include")]

    def one(src):
        obj = os.path.join(odir, os.path.basename(src) + ".o")
        return subprocess.run([*base, "-c", "-o", obj, src], capture_output=True, text=True), obj

    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
        results = list(ex.map(one, sources()))
    log = "".join(r.stderr for r, _ in results)
    bad = [r for r, _ in results if r.returncode != 0]
    if bad:
        sys.stderr.write("".join(r.stdout + r.stderr for r in bad))
        raise RuntimeError(f"nvcc failed building {os.path.basename(out)}")
    link = subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                           "-o", out + ".tmp", *[o for _, o in results]],
                          capture_output=True, text=True)
    if link.returncode != 0:
        sys.stderr.write(link.stdout + link.stderr)
        raise RuntimeError(f"nvcc failed linking {os.path.basename(out)}")
    os.replace(out + ".tmp", out)
    return log


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    log = _compile(LIB, [])
    with open(os.path.join(HERE, "csrc", "ptxas_report.txt"), "w") as f:
        f.write(log)
    if verbose:
        sys.stderr.write(log)
    return LIB


def build_variant(name: str, defines: list[str]) -> str:
    """Development aid: the library with extra -D flags into build/variants/
    (selected at import with GWN_B200_LIB=<path>); not used by the product."""
    out = os.path.join(REPO, "build", "variants", f"libgwn_b200_{name}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    _compile(out, defines)
    return out


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--variant":
        print(build_variant(sys.argv[2], sys.argv[3:]))
    else:
        print(build(force="--force" in sys.argv, verbose=True))
