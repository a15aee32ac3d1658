"""Drop-in ``caqr.caqr`` -> paper_0809_2407_b200.caqr."""
from paper_0809_2407_b200.caqr import *  # noqa: F401,F403
from paper_0809_2407_b200 import caqr as _impl

globals().update({k: getattr(_impl, k) for k in dir(_impl) if not k.startswith("__")})
