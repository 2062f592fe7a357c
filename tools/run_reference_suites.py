"""Run the reference's own test suites (/root/reference/pkg/tests) unmodified against this
package imported as ``sikv`` (paper_2603_14224_b200/compat/sikv: numpy in / numpy out over the
B200 implementation).

    python tools/run_reference_suites.py --stage      # here: copy the suites to baseline/_ref/pkg_tests
    python tools/run_reference_suites.py [pytest args] # on the GPU box: run them

baseline/_ref/ is git-ignored (the reference is never committed) but travels to the GPU box with
the repo snapshot; the suites are test code of the reference, run as-is.
"""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEST = os.path.join(ROOT, "baseline", "_ref", "pkg_tests")
SRC = "/root/reference/pkg/tests"

if "--stage" in sys.argv:
    os.makedirs(DEST, exist_ok=True)
    for f in sorted(os.listdir(SRC)):
        if f.endswith(".py"):
            shutil.copy(os.path.join(SRC, f), os.path.join(DEST, f))
    print(f"staged {len(os.listdir(DEST))} files in {DEST}")
    sys.exit(0)

env = dict(os.environ)
env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "paper_2603_14224_b200", "compat"), ROOT,
                                     env.get("PYTHONPATH", "")])
args = sys.argv[1:] or ["-q"]
sys.exit(subprocess.call([sys.executable, "-m", "pytest", DEST, "-p", "no:cacheprovider", "--rootdir", DEST, *args],
                         env=env, cwd=DEST))
