"""``import dbsim`` -> the B200 implementation.

The reference ships its API as the pure-Python package ``dbsim``
(pkg/src/dbsim/__init__.py:15-63).  This alias makes the drop-in literal: code
written against ``dbsim`` (including the reference's own test-suite, run as the
API-conformance suite in tests/ref_conformance/) imports
``paper_2007_11831_b200`` unchanged -- same names, same exception classes, same
submodules (allocation, cluster, sgdlab, checks, report, errors), every numeric
step on the sm_100a kernels.  ``dbsim.scenarios`` / ``dbsim.cli`` (YAML configs
and the command-line runner) are out of the hot-path scope and are
not provided.
"""

import sys as _sys

import paper_2007_11831_b200 as _impl
from paper_2007_11831_b200 import *  # noqa: F401,F403
from paper_2007_11831_b200 import allocation, checks, cluster, errors, report, sgdlab  # noqa: F401

for _name in ("allocation", "checks", "cluster", "errors", "report", "sgdlab"):
    _sys.modules[f"{__name__}.{_name}"] = getattr(_impl, _name)

__version__ = getattr(_impl, "__version__", "0.1.0")
