"""Build libfdfb.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build()."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "fdfb_api.cu")
OUT = os.path.join(HERE, "libfdfb.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUDA_LIB = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "lib64")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr", "-Xptxas", "-v",
         "-L" + CUDA_LIB, "-Xlinker", "-rpath=" + CUDA_LIB]


def sources():
    d = os.path.join(HERE, "csrc")
    return [os.path.join(d, f) for f in os.listdir(d)] + [os.path.join(os.path.dirname(HERE), "include", "fdfb.h")]


HASH = OUT + ".srchash"


def source_hash() -> str:
    import hashlib
    h = hashlib.sha256()
    for s in sorted(sources()):
        if s.endswith((".cu", ".cuh", ".inc", ".h")):
            h.update(os.path.basename(s).encode())
            with open(s, "rb") as f:
                h.update(f.read())
    return h.hexdigest()


def is_stale() -> bool:
    """True if libfdfb.so was not built from the current sources (content hash, not mtimes)."""
    if not os.path.exists(OUT) or not os.path.exists(HASH):
        return True
    with open(HASH) as f:
        return f.read().strip() != source_hash()


def needs_build() -> bool:
    return is_stale()


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libfdfb.so if stale.  Concurrent callers (torchrun ranks) serialise on a file
    lock; nvcc writes a temporary file that replaces the library atomically, so no process
    ever maps a half-written .so, and a process that waited finds it fresh and skips."""
    import fcntl
    if not (force or needs_build()):
        return OUT
    with open(OUT + ".lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        try:
            if force or needs_build():
                tmp = "%s.tmp.%d" % (OUT, os.getpid())
                cmd = [NVCC] + FLAGS + ["-o", tmp, SRC]
                r = subprocess.run(cmd, capture_output=True, text=True)
                log = os.path.join(HERE, "build.log")
                with open(log, "w") as f:
                    f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
                if r.returncode != 0:
                    if os.path.exists(tmp):
                        os.remove(tmp)
                    sys.stderr.write(r.stderr[-6000:])
                    raise RuntimeError("nvcc failed (see %s)" % log)
                os.replace(tmp, OUT)
                with open(HASH + ".tmp", "w") as f:
                    f.write(source_hash())
                os.replace(HASH + ".tmp", HASH)
                if verbose:
                    sys.stderr.write(r.stderr)
        finally:
            fcntl.flock(lk, fcntl.LOCK_UN)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
