"""Per-step latency phases of the sorted construction kernel (clock64 probes).

Build the instrumented library and run on a GPU:
    python scripts/step_profile.py --build      (here: nvcc -DTACO_STEP_PROFILE)
    TACO_LIB_PATH=build/libtaco_prof.so python scripts/step_profile.py --m 512
"""
import argparse
import ctypes
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "build", "libtaco_prof.so")

ap = argparse.ArgumentParser()
ap.add_argument("--build", action="store_true")
ap.add_argument("--n", type=int, default=2392)
ap.add_argument("--m", type=int, default=512)
args = ap.parse_args()
if args.build:
    srcs = sorted(glob.glob(os.path.join(ROOT, "paper_2404_04895_b200", "csrc", "*.cu")))
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                    "-Xcompiler", "-fPIC", "-shared", "-DTACO_STEP_PROFILE", "-I", os.path.join(ROOT, "include"),
                    "-o", OUT, *srcs], check=True)
    print(OUT)
    sys.exit(0)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2404_04895_b200 as taco  # noqa: E402
from paper_2404_04895_b200 import _device, _lib  # noqa: E402

lib = _lib.load()
lib.taco_step_profile.argtypes = [ctypes.c_void_p, ctypes.c_int]
inst = taco.euclidean_instance(np.random.default_rng(0).uniform(0, 2000, (args.n, 2)))
params = taco.AcoParams(m=args.m, k=max(1, args.m // 10), selection="adair", seed=0)
s = taco.Solver(inst, params)
for _ in range(3):
    s.step_async()
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
lib.taco_step_profile(buf, 1)
s.step_async()
torch.cuda.synchronize()
lib.taco_step_profile(buf, 0)
steps = buf[3]
print({"m": args.m, "steps": steps, "global_cycles": buf[1] / steps,
       "bookkeeping_cycles": buf[2] / steps, "global_windows_per_step": buf[4] / steps,
       "first_window_load_wait": buf[5] / steps, "vis_philox_key_cycles": buf[6] / steps,
       "two_redux_cycles": buf[7] / steps})
