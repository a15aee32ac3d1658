"""Drop-in ``caqr.tsqr`` -> paper_0809_2407_b200.tsqr (see package docstring)."""
from paper_0809_2407_b200.tsqr import *  # noqa: F401,F403
from paper_0809_2407_b200 import tsqr as _impl

globals().update({k: getattr(_impl, k) for k in dir(_impl) if not k.startswith("__")})
