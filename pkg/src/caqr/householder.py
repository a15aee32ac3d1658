"""Drop-in ``caqr.householder`` -> paper_0809_2407_b200.householder (see package docstring)."""
from paper_0809_2407_b200.householder import *  # noqa: F401,F403
from paper_0809_2407_b200 import householder as _impl

globals().update({k: getattr(_impl, k) for k in dir(_impl) if not k.startswith("__")})
