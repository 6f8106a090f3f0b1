"""Build libsimplicial_trace.so (relocatable device code, -DSA_TRACE) for phase timelines."""
import glob, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2507_02754_b200", "csrc")
OUT = os.path.join(ROOT, "paper_2507_02754_b200", "libsimplicial_trace.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
objs = []
for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
    obj = f"/tmp/trace_{os.path.basename(src)}.o"
    subprocess.check_call(["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-rdc=true", "-DSA_TRACE", *os.environ.get("SA_EXTRA", "").split(),
                           "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-c", src, "-o", obj])
    objs.append(obj)
subprocess.check_call(["nvcc", *ARCH, "-shared", "-rdc=true", "-o", OUT, *objs])
print(OUT)
