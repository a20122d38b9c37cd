"""In-tree build of the native libraries (sm_100a only).

    lib/libacg.so        the product: C ABI of include/acg.h (host automaton + CUDA scan)
    lib/libacg_synth.so  deterministic synthetic corpora for the BASELINE workloads

Run `python -m paper_1403_7294_b200.native` (or __graft_entry__.build()).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


HOST_SOURCES = ("automaton.cpp", "parallel.cpp", "host_io.cpp")  # host C++ of libacg.so
DEVICE_SOURCES = ("acg_device.cu",)  # CUDA translation units of libacg.so


def build(force: bool = False, verbose_ptxas: bool = False) -> None:
    os.makedirs(LIB, exist_ok=True)
    obj = os.path.join(LIB, "obj")
    os.makedirs(obj, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include")]

    synth = os.path.join(LIB, "libacg_synth.so")
    src = os.path.join(CSRC, "synth.cpp")
    if force or _stale(synth, [src]):
        _run(["g++", "-std=c++17", "-O3", "-fPIC", "-shared", "-pthread", "-o", synth, src])

    headers = [os.path.join(CSRC, h) for h in ("automaton.hpp", "scan_kernels.cuh", "filter_kernels.cuh",
                                               "exact_kernels.cuh", "format_kernels.cuh", "partition.cuh", "qfilter.hpp", "ctab.hpp", "parallel.hpp")] + [
        os.path.join(ROOT, "include", "acg.h")]
    host_objs = []
    for name in HOST_SOURCES:
        src_c = os.path.join(CSRC, name)
        o = os.path.join(obj, name.replace(".cpp", ".o"))
        if force or _stale(o, [src_c] + headers):
            _run(["g++", "-std=c++17", "-O3", "-fPIC", "-pthread", "-c", "-o", o, src_c] + inc +
                 ["-I", os.path.join(os.path.dirname(NVCC), "..", "include")])
        host_objs.append(o)
    dev_objs = []
    for name in DEVICE_SOURCES:
        dev_src = os.path.join(CSRC, name)
        dev_o = os.path.join(obj, name.replace(".cu", ".o"))
        if force or _stale(dev_o, [dev_src] + headers):
            cmd = [NVCC, *ARCH, "-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-c", "-o", dev_o, dev_src] + inc
            if verbose_ptxas:
                cmd.insert(1, "-Xptxas=-v")
            _run(cmd)
        dev_objs.append(dev_o)
    lib = os.path.join(LIB, "libacg.so")
    if force or _stale(lib, host_objs + dev_objs):
        _run([NVCC, *ARCH, "-shared", "-o", lib, *host_objs, *dev_objs, "-Xcompiler", "-pthread"])


def build_variant(name: str, defines: list[str]) -> str:
    """Experiment builds (kernel ablations) into lib/variants/<name>/libacg.so."""
    out = os.path.join(LIB, "variants", name)
    os.makedirs(out, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include")]
    dev_o = os.path.join(out, "acg_device.o")
    _run([NVCC, *ARCH, "-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-c", "-o", dev_o,
          os.path.join(CSRC, "acg_device.cu")] + inc + [f"-D{d}" for d in defines])
    lib = os.path.join(out, "libacg.so")
    host_objs = [os.path.join(LIB, "obj", name.replace(".cpp", ".o")) for name in HOST_SOURCES]
    others = [os.path.join(LIB, "obj", name.replace(".cu", ".o")) for name in DEVICE_SOURCES if name != "acg_device.cu"]
    _run([NVCC, *ARCH, "-shared", "-o", lib, *host_objs, dev_o, *others, "-Xcompiler", "-pthread"])
    return lib


def build_oracle() -> None:
    """Test infrastructure: the C restatement and (when /root/reference is
    present) the reference compiled into oracle/_ref/."""
    _run(["make", "-s", "-C", os.path.join(ROOT, "oracle")])


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)
    build_oracle()
