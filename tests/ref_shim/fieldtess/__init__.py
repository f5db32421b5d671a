"""Import shim: the reference's test suite imports ``fieldtess``; this
package answers with paper_1804_09152_b200 (the drop-in under test), its
submodules registered under the reference's module names."""

import sys

import paper_1804_09152_b200 as _impl
from paper_1804_09152_b200 import *  # noqa: F401,F403
from paper_1804_09152_b200 import analysis, dual, errors, field, lloyd, mesh, sparse  # noqa: F401

for _name in ("analysis", "dual", "errors", "field", "lloyd", "mesh", "sparse"):
    sys.modules[f"{__name__}.{_name}"] = getattr(_impl, _name)

__version__ = _impl.__version__
