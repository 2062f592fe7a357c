"""Analytic operation counters (reference: sikv/instrument.py)."""
from .api import OpCounters, collect, tally  # noqa: F401
