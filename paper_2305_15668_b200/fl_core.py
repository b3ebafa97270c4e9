"""Module alias so `from paper_2305_15668_b200.fl_core import X` works like `from fedsim.fl_core import X`."""

from .training import *  # noqa: F401,F403
from . import training as _impl

globals().update({k: v for k, v in vars(_impl).items() if not k.startswith("__")})
