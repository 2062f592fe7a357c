"""The reference's own test suites (/root/reference/pkg/tests: normalize, codebook, quantizer,
retrieval, attention, cache, acceptance c01-c10, bench, cli, synth, tensorfile), unmodified,
against this package imported as ``sikv`` (paper_2603_14224_b200/compat/sikv).

The suites are staged (git-ignored) into baseline/_ref/pkg_tests by
``python tools/run_reference_suites.py --stage`` in the build container; the staged copy
travels to the GPU box with the repo snapshot."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGED = os.path.join(ROOT, "baseline", "_ref", "pkg_tests")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.isdir(STAGED), reason="reference suites not staged (tools/run_reference_suites.py --stage)")
def test_reference_suites_pass_unmodified():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "run_reference_suites.py"), "-q"],
                       capture_output=True, text=True, timeout=1800)
    tail = "\n".join(r.stdout.strip().splitlines()[-15:])
    assert r.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail, tail
