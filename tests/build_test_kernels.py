"""Build the test-only cuRAND Philox reference library (tests/_curand_ref.so)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cuda", "curand_philox_ref.cu")
OUT = os.path.join(HERE, "_curand_ref.so")


def build() -> str:
    if os.path.exists(OUT) and os.path.getmtime(OUT) >= os.path.getmtime(SRC):
        return OUT
    cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2",
           "-Xcompiler", "-fPIC", "-shared", SRC, "-o", OUT]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(r.stderr)
    return OUT


if __name__ == "__main__":
    print(build())
