"""Build libee.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels
to the GPU box with the repo snapshot)."""
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libee.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(HERE, "..", "include", "*.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force=False, verbose=False, trace=False, variant=None, defines=()):
    """trace=True: the profiling variant libee_trace.so (-DEE_TRACE timeline
    probes, tools/attn_timeline.py); variant="name" with `defines` builds an
    A/B copy libee_<name>.so (loaded through EE_LIB_PATH by the timing tools).
    Neither is ever loaded by the product path."""
    name = "trace" if trace else variant
    target = OUT.replace("libee.so", f"libee_{name}.so") if name else OUT
    if not force and not name and not needs_build():
        return OUT
    objdir = os.path.join(HERE, f"build_{name}" if name else "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    log = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *FLAGS, *(["-DEE_TRACE"] if trace else []), *defines, "-c", src, "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    for cmd, p in procs:
        out, _ = p.communicate()
        log.append(out.decode())
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", target + ".tmp"]
    subprocess.check_call(cmd)
    os.replace(target + ".tmp", target)
    with open(os.path.join(objdir, "ptxas.log"), "w") as f:
        f.write("\n".join(log))
    if verbose:
        print("\n".join(log))
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv))
