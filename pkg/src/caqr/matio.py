"""Drop-in ``caqr.matio`` -> paper_0809_2407_b200.matio (see package docstring)."""
from paper_0809_2407_b200.matio import *  # noqa: F401,F403
from paper_0809_2407_b200 import matio as _impl

globals().update({k: getattr(_impl, k) for k in dir(_impl) if not k.startswith("__")})
