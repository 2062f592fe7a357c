"""``sikv`` alias of the B200 implementation (host-array API: paper_2603_14224_b200.hostapi).
The reference's test suites run against it unmodified (tools/run_reference_suites.py)."""
from paper_2603_14224_b200.hostapi import *  # noqa: F401,F403
from paper_2603_14224_b200.hostapi import __all__  # noqa: F401

__version__ = "0.1.0"
