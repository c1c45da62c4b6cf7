"""ORACLE -- TEST INFRASTRUCTURE ONLY.

A CPU restatement of the reference `pforvec` execution path (its NumPy kernel
library and its executor, including the per-iteration SIMD interpreter), run
in float64 exactly like the reference.  It is the checker for the B200 path
and the timed CPU baseline in bench.py; it is never imported by the product
package.  Parity of this restatement with the reference itself is pinned by
the golden fixtures in tests/golden/ (made by tests/golden/make_golden.py,
which imports the real reference from /root/reference in the build container).
"""

from .executor import OracleExecutor, RngState, VariableStore, execute  # noqa: F401
from . import kernels  # noqa: F401
