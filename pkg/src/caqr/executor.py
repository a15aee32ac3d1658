"""Drop-in ``caqr.executor`` -> paper_0809_2407_b200.executor (see package docstring)."""
from paper_0809_2407_b200.executor import *  # noqa: F401,F403
from paper_0809_2407_b200 import executor as _impl

globals().update({k: getattr(_impl, k) for k in dir(_impl) if not k.startswith("__")})
