"""Drop-in ``caqr.core`` -> paper_0809_2407_b200.core (see package docstring)."""
from paper_0809_2407_b200.core import *  # noqa: F401,F403
from paper_0809_2407_b200 import core as _impl

globals().update({k: getattr(_impl, k) for k in dir(_impl) if not k.startswith("__")})
