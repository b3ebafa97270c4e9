"""Module alias so `from paper_2305_15668_b200.profiles import X` works like `from fedsim.profiles import X`."""

from .spec import *  # noqa: F401,F403
from . import spec as _impl

globals().update({k: v for k, v in vars(_impl).items() if not k.startswith("__")})
