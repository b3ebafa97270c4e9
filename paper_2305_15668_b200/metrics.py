"""Module alias so `from paper_2305_15668_b200.metrics import X` works like `from fedsim.metrics import X`."""

from .roundsim import *  # noqa: F401,F403
from . import roundsim as _impl

globals().update({k: v for k, v in vars(_impl).items() if not k.startswith("__")})
from .roundsim import KIND_RANK  # noqa: E402,F401
