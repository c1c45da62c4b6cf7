"""Exception hierarchy.

The class names are part of the drop-in contract: callers of the reference
catch these by name (reference `pkg/src/pforvec/errors.py:1-127`), so the B200
executor raises the same classes -- host-side validation raises them before a
launch, and device error words are mapped back onto them after a sync.
"""

from __future__ import annotations


class PforVecError(Exception):
    """Root of every error this package raises."""


def _simple(name: str, doc: str):
    return type(name, (PforVecError,), {"__doc__": doc})


# kernel-level validation (reference errors.py:10-43)
IncompatibleShapes = _simple("IncompatibleShapes", "Shapes cannot be combined.")
DTypeMismatch = _simple("DTypeMismatch", "Operand dtypes are not accepted by the op.")
RankError = _simple("RankError", "Operand rank is not accepted by the op.")
AxisOutOfRange = _simple("AxisOutOfRange", "Axis outside [-rank, rank).")
DuplicateAxis = _simple("DuplicateAxis", "An axis appears twice after normalisation.")
IndexOutOfBounds = _simple("IndexOutOfBounds", "Row index outside [0, n).")
IndexCollision = _simple("IndexCollision", "Two index sets write the same row.")
IncompleteCover = _simple("IncompleteCover", "Index sets leave rows unwritten.")
BadPermutation = _simple("BadPermutation", "Transpose perm is not a permutation.")

# graph construction (reference errors.py:48-74)
UnknownInput = _simple("UnknownInput", "Input ref does not resolve in this graph.")
BadAttr = _simple("BadAttr", "Node attributes are missing, extra or malformed.")
ArityMismatch = _simple("ArityMismatch", "Branch/body output counts disagree.")
NonScalarCondition = _simple("NonScalarCondition", "cond predicate is not a bool scalar.")


class CycleDetected(PforVecError):
    def __init__(self, msg, nodes=()):
        super().__init__(msg)
        self.nodes = tuple(nodes)


class ParseError(PforVecError):
    def __init__(self, msg, line, col):
        super().__init__(f"{msg} at line {line}, column {col}")
        self.line = line
        self.col = col


# execution (reference errors.py:79-93)
class ExecError(PforVecError):
    """An op failed; `node_id` names the graph node, `cause` the kernel error."""

    def __init__(self, node_id, cause):
        super().__init__(f"node {node_id}: {cause}")
        self.node_id = node_id
        self.cause = cause


ShapeVariance = _simple("ShapeVariance", "Per-iteration outputs disagree in shape.")
BudgetExceeded = _simple("BudgetExceeded", "Dispatch budget exhausted.")

# vectorizer / autodiff (reference errors.py:98-117)
VectorizeError = _simple("VectorizeError", "The body cannot be converted.")
StatefulNotSupported = type("StatefulNotSupported", (VectorizeError,),
                            {"__doc__": "Stateful op has no SIMD-compatible form."})
NonScalarOutput = _simple("NonScalarOutput", "gradient() of a non-scalar without a seed.")
NonDifferentiableOp = _simple("NonDifferentiableOp", "No VJP rule applies.")
ShapeMismatch = _simple("ShapeMismatch", "Gradient shape mismatch.")

# device runtime (new: the native layer's failure modes)
NativeUnavailable = _simple(
    "NativeUnavailable",
    "The sm_100a kernel library is not built/loadable or no CUDA device is present. "
    "There is deliberately no CPU fallback.")
DeviceError = _simple("DeviceError", "A CUDA API call or kernel launch failed.")
