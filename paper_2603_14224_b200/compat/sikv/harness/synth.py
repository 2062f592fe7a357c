"""sikv.harness.synth alias."""
from paper_2603_14224_b200.harness.synth import *  # noqa: F401,F403
from paper_2603_14224_b200.harness import synth as _m

globals().update({k: v for k, v in vars(_m).items() if not k.startswith('__')})
