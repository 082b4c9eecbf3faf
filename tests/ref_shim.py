"""pytest plugin: run the REFERENCE's own test suite on the B200 kernel.

Loaded with ``-p ref_shim`` before the reference package is imported, it
installs paper_2605_19926_b200.tilecast_backend (the drop-in backend over the
C ABI) as ``tilecast.backend._core`` -- the module the reference's backend
selector imports for "compiled" (backend/__init__.py:20-25). The reference's
cross-backend tests then compare the CUDA kernel with its own pure-Python
kernels bit for bit.
"""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_2605_19926_b200 import tilecast_backend  # noqa: E402

sys.modules["tilecast.backend._core"] = tilecast_backend
