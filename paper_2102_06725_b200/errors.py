"""Exception hierarchy of the drop-in API.

The class names (and their base, ``NnlError``) are the reference's public
error vocabulary (reference ``src/errors.py:8-122``); code that catches
``nanonnl`` errors catches these unchanged.  The native library reports
failures as integer status codes (include/nnl.h) which ``_lib`` maps back
onto the same classes.
"""

from __future__ import annotations


class NnlError(Exception):
    """Root of every error raised on purpose by this package."""


def _kind(name: str, doc: str, base: type = NnlError) -> type:
    return type(name, (base,), {"__doc__": doc, "__module__": __name__})


# array / kernel level
ShapeMismatch = _kind("ShapeMismatch", "Operand shapes are incompatible.")
InvalidRange = _kind("InvalidRange", "A numeric range is empty or inverted.")
KernelTooLarge = _kind("KernelTooLarge", "A window exceeds the padded input extent.")
# (extension) a device kernel computes in one storage type: operands whose
# dtypes disagree are refused at apply() instead of being misread
DtypeMismatch = _kind("DtypeMismatch", "Operand storage dtypes are incompatible.", ShapeMismatch)
# graph level
UnknownFunction = _kind("UnknownFunction", "No function kind of that name is registered.")
CycleDetected = _kind("CycleDetected", "Graph traversal found a cycle.")
UninitializedInput = _kind("UninitializedInput", "A leaf was read before data was assigned.")
ForwardNotRun = _kind("ForwardNotRun", "backward ran before forward produced activations.")
LabelOutOfRange = _kind("LabelOutOfRange", "A label lies outside [0, num_classes).")
DegenerateBatch = _kind("DegenerateBatch", "Batch statistics over a single element.")
# parameters
ShapeConflict = _kind("ShapeConflict", "A registry name already exists with another shape.")
# solver
EmptyParameterSet = _kind("EmptyParameterSet", "Solver setup received no parameters.")
NotSetup = _kind("NotSetup", "A solver method was called before setup().")
# communicator
InvalidWorkerCount = _kind("InvalidWorkerCount", "Worker count must be >= 1 and divide the batch.")
ShapeMismatchAcrossRanks = _kind("ShapeMismatchAcrossRanks", "Ranks disagree on buffer lists.")
CollectiveTimeout = _kind("CollectiveTimeout", "A rank failed to join a collective in time.")
DivergedReplicas = _kind("DivergedReplicas", "Replica parameters differ after a step.")


class DeviceError(NnlError):
    """The native library reported a CUDA or configuration failure."""


__all__ = [
    "NnlError", "ShapeMismatch", "InvalidRange", "KernelTooLarge", "DtypeMismatch", "UnknownFunction",
    "CycleDetected", "UninitializedInput", "ForwardNotRun", "LabelOutOfRange",
    "DegenerateBatch", "ShapeConflict", "EmptyParameterSet", "NotSetup",
    "InvalidWorkerCount", "ShapeMismatchAcrossRanks", "CollectiveTimeout",
    "DivergedReplicas", "DeviceError",
]
