"""Build a libmask variant with extra -D flags into tools/variants/<name>.so (A/B timing)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_02734_b200 import buildlib

def build(name, defines):
    inc, libdir = buildlib._nccl_dirs()
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "variants")
    os.makedirs(out, exist_ok=True)
    objs, procs = [], []
    for s in buildlib.sources():
        o = f"/tmp/var_{name}_" + os.path.basename(s).replace(".cu", ".o")
        cmd = [buildlib.NVCC, "-c", s, "-o", o] + buildlib.ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler",
               "-fPIC", "-I", inc, "-I", os.path.join(buildlib.ROOT, "include"), "--expt-relaxed-constexpr"] + \
              [f"-D{d}" for d in defines]
        procs.append(subprocess.Popen(cmd))
        objs.append(o)
    for p in procs:
        assert p.wait() == 0
    so = os.path.join(out, name + ".so")
    subprocess.check_call([buildlib.NVCC, "-shared", "-o", so] + objs + buildlib.ARCH +
                          ["-cudart", "static", "-L", libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + libdir])
    return so

if __name__ == "__main__":
    print(build(sys.argv[1], sys.argv[2:]))
