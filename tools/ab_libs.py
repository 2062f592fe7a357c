"""A/B timing of alternative in-tree builds (SIKV_LIB=<name>.so each, built with
SIKV_BUILD_SUFFIX / SIKV_NVCC_EXTRA): runs kernel_ab.py for every library, alternating, R rounds.
    python tools/ab_libs.py "libsikv_b200.so libsikv_x.so" c2 c4   [env KERNELS, R]"""
import os
import subprocess
import sys

libs = sys.argv[1].split()
cfgs = sys.argv[2:] or ["c2"]
here = os.path.dirname(os.path.abspath(__file__))
for r in range(int(os.environ.get("R", "2"))):
    for lib in libs:
        env = dict(os.environ, SIKV_LIB=lib)
        out = subprocess.run([sys.executable, os.path.join(here, "kernel_ab.py"), *cfgs], env=env,
                             capture_output=True, text=True)
        for line in (out.stdout + out.stderr).strip().splitlines():
            print(f"[{lib}] {line}", flush=True)
