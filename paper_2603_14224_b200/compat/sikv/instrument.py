"""sikv.instrument alias."""
from paper_2603_14224_b200.instrument import OpCounters, collect, tally  # noqa: F401
