"""Drop-in ``caqr.trees`` -> paper_0809_2407_b200.trees (see package docstring)."""
from paper_0809_2407_b200.trees import *  # noqa: F401,F403
from paper_0809_2407_b200 import trees as _impl

globals().update({k: getattr(_impl, k) for k in dir(_impl) if not k.startswith("__")})
