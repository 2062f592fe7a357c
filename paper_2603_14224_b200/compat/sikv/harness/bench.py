"""sikv.harness.bench alias."""
from paper_2603_14224_b200.harness.bench import *  # noqa: F401,F403
from paper_2603_14224_b200.harness import bench as _m

globals().update({k: v for k, v in vars(_m).items() if not k.startswith('__')})
