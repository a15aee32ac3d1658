"""Drop-in ``caqr`` package (reference: pkg/src/caqr, SPEC.md) backed by the
B200-native implementation in ``paper_0809_2407_b200``.

The reference's modules keep their names: ``caqr.core``, ``caqr.trees``,
``caqr.counters``, ``caqr.executor``, ``caqr.householder`` and the SPEC's
``caqr.tsqr`` / ``caqr.caqr``.  Put ``pkg/src`` on ``sys.path`` (or install
this directory) in place of the reference's ``pkg/src``.
"""
import os as _os
import sys as _sys

_ROOT = _os.path.dirname(_os.path.dirname(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__)))))
if _ROOT not in _sys.path:
    _sys.path.insert(0, _ROOT)
