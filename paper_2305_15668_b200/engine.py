"""Module alias so `from paper_2305_15668_b200.engine import X` works like `from fedsim.engine import X`."""

from .experiment import *  # noqa: F401,F403
from . import experiment as _impl

globals().update({k: v for k, v in vars(_impl).items() if not k.startswith("__")})
from .roundsim import run_round  # noqa: E402,F401
