"""sikv.harness.cli alias."""
from paper_2603_14224_b200.harness.cli import *  # noqa: F401,F403
from paper_2603_14224_b200.harness import cli as _m

globals().update({k: v for k, v in vars(_m).items() if not k.startswith('__')})
