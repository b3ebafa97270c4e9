"""Module alias so `from paper_2305_15668_b200.scheduler import X` works like `from fedsim.scheduler import X`."""

from .planner import *  # noqa: F401,F403
from . import planner as _impl

globals().update({k: v for k, v in vars(_impl).items() if not k.startswith("__")})
