"""pytest plugin (``-p coesim_shim``): make ``import coesim`` load the shim in
``tests/shim/coesim`` (this package under the reference's name)."""

import coesim  # noqa: F401
