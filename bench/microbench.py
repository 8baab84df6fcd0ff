"""Build/run the L0 microbenchmark (bench/microbench.cu)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "microbench.cu")
BIN = os.path.join(HERE, "microbench")


def build():
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < os.path.getmtime(SRC):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
                               "-std=c++17", "-o", BIN, SRC])
    return BIN


if __name__ == "__main__":
    build()
    subprocess.check_call([BIN])
