"""Build liblinksim_b200.so (sm_100a) in-tree with nvcc.

Used by __graft_entry__.build() and `python -m paper_2203_11854_b200._build`.
Each .cu compiles to its own object in parallel, then one shared library is
linked next to this file so it travels with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "liblinksim_b200.so")
SOURCES = ["capi.cu", "bp_exact.cu", "bp_fast.cu", "rng_normal.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wshadow",
         "-I", os.path.join(ROOT, "include")]


GEN = os.path.join(ROOT, "build", "gen")
# per-source extra flags: the numpy-replica RNG must round every operation
# separately, as the host libm/numpy code it mirrors does
EXTRA = {"rng_normal.cu": ["-fmad=false"]}
# the exact decoders reproduce numpy's separately rounded f64 operations
EXTRA_PREFIX = {"qcx_": ["-fmad=false"]}


def _instance_sources():
    """One translation unit per specialised fast-decoder instance listed in
    csrc/qc_instances.h, so they compile in parallel."""
    import re

    text = open(os.path.join(CSRC, "qc_instances.h")).read()
    os.makedirs(GEN, exist_ok=True)
    out = []
    for bg, z, r, sp, pr in re.findall(r"X\((\d+),\s*(\d+),\s*(\d+),\s*(\d+),\s*(\w+)\)", text):
        name = f"qc_{pr}_{bg}_{z}_{r}.cu"
        launcher = {"f32": "launch_qc_fast2", "h2": "launch_qc_fast_h2", "sp": "launch_qc_sp",
                    "sp32": "launch_qc_sp32"}[pr]
        body = (f'#include "{CSRC}/bp_fast_h2.cuh"\n#include "{CSRC}/bp_fast_sp.cuh"\n'
                "namespace lsb {\n"
                f"int qc2_{pr}_{bg}_{z}_{r}(const QcChanParams &P, const float *l, int64_t B, int it, float a, int es,\n"
                "    uint8_t *h, float *lo, int32_t *iu, const uint8_t *ref, unsigned long long *cnt, cudaStream_t s) {\n"
                f"  return {launcher}<BG{bg}Tables, {z}, {r}, {sp}>(P, l, B, it, a, es, h, lo, iu, ref, cnt, s);\n"
                "}\n}  // namespace lsb\n")
        out.append(_write(name, body))
    for bg, rb, sp in re.findall(r"Y\((\d+),\s*(\d+),\s*(\d+)\)", text):
        body = (f'#include "{CSRC}/bp_fast_h2.cuh"\n'
                "namespace lsb {\n"
                f"int qcrt_{bg}_{rb}_{sp}(const QcChanParams &P, int R, const uint16_t *s, const int32_t *col,\n"
                "    const float *l, int64_t B, int it, float a, int es, uint8_t *h, float *lo, int32_t *iu,\n"
                "    const uint8_t *ref, unsigned long long *cnt, cudaStream_t st) {\n"
                f"  return launch_qc_h2rt<BG{bg}Tables, {rb}, {sp}>(P, R, s, col, l, B, it, a, es, h, lo, iu, ref, cnt, st);\n"
                "}\n}  // namespace lsb\n")
        out.append(_write(f"qcrt_{bg}_{rb}_{sp}.cu", body))
    for bg, rb, sp in re.findall(r"W\((\d+),\s*(\d+),\s*(\d+)\)", text):
        body = (f'#include "{CSRC}/bp_fast_sp.cuh"\n'
                "namespace lsb {\n"
                f"int qcsprt_{bg}_{rb}_{sp}(const QcChanParams &P, int R, const uint16_t *s, const int32_t *col,\n"
                "    const float *l, int64_t B, int it, float a, int es, uint8_t *h, float *lo, int32_t *iu,\n"
                "    const uint8_t *ref, unsigned long long *cnt, cudaStream_t st) {\n"
                f"  return launch_qc_sprt<BG{bg}Tables, {rb}, {sp}>(P, R, s, col, l, B, it, a, es, h, lo, iu, ref, cnt, st);\n"
                "}\n}  // namespace lsb\n")
        out.append(_write(f"qcsprt_{bg}_{rb}_{sp}.cu", body))
    for bg, z, ntl in re.findall(r"V\((\d+),\s*(\d+),\s*(\d+)\)", text):
        for mt, tag in (("double", "qcx"), ("float", "qcf")):
            body = (f'#include "{CSRC}/bp_qc_exact.cuh"\n'
                    "namespace lsb {\n"
                    f"int {tag}_{bg}_{z}(const QcChanParams &P, const float *l, int64_t B, int it, double a, int es,\n"
                    "    int mo, uint8_t *h, int hl, float *lo, int32_t *iu, const uint8_t *ref,\n"
                    "    unsigned long long *cnt, cudaStream_t s) {\n"
                    f"  return launch_qc_exact<BG{bg}Tables, {z}, {ntl}, {mt}>(P, l, B, it, a, es, mo, h, hl, lo, iu, ref,\n"
                    "                                                          cnt, s);\n"
                    "}\n}  // namespace lsb\n")
            out.append(_write(f"{tag}_{bg}_{z}.cu", body))
    return out


def _write(name: str, body: str) -> str:
    path = os.path.join(GEN, name)
    if not os.path.exists(path) or open(path).read() != body:
        with open(path, "w") as f:
            f.write(body)
    return path




def _deps(path: str, seen=None) -> set:
    """The file and every local header it includes, recursively."""
    import re

    seen = set() if seen is None else seen
    if path in seen or not os.path.exists(path):
        return seen
    seen.add(path)
    for inc in re.findall(r'^\s*#\s*include\s+"([^"]+)"', open(path).read(), re.M):
        _deps(os.path.normpath(os.path.join(os.path.dirname(path), inc)), seen)
    return seen


def _compile(src: str, verbose: bool, newest_hdr: float, force: bool) -> str:
    obj = os.path.join(OBJ, os.path.splitext(os.path.basename(src))[0] + ".o")
    newest_dep = max(os.path.getmtime(f) for f in _deps(src))
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep:
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, *EXTRA.get(os.path.basename(src), []),
           *[f for p, fl in EXTRA_PREFIX.items() if os.path.basename(src).startswith(p) for f in fl], "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose:
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    sys.path.insert(0, ROOT)
    from tools import gen_bg_header

    gen_bg_header.main()
    srcs = [os.path.join(CSRC, f) for f in SOURCES] + _instance_sources()
    hdrs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    hdrs.append(os.path.join(ROOT, "include", "linksim_b200.h"))
    newest_hdr = max(os.path.getmtime(f) for f in hdrs)
    newest = max(newest_hdr, max(os.path.getmtime(f) for f in srcs))
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= newest:
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    with concurrent.futures.ThreadPoolExecutor(min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, newest_hdr, force), srcs))
    tmp = LIB + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
