"""Exception taxonomy of the reference, raised from C-ABI status codes.

Each class carries the name of the reference exception it stands for, so
code written against ``seqlab`` catches the same types.
"""


class ShardError(ValueError):
    """An axis cannot be split evenly across the group (simgroup.py:62-63)."""


class DivisibilityError(ValueError):
    """A dimension is not divisible by the partition count (tensor.py:27-28)."""


class GroupDesyncError(RuntimeError):
    """Ranks diverged: inconsistent collective arguments or a timeout
    (simgroup.py:66-67).  Never a hang: device waits are bounded."""


class KernelError(ValueError):
    """Kernel and mask/dtype/head_dim are incompatible (kernels.py:22-23)."""


class ForwardStateError(ValueError):
    """Backward called without a matching saved forward state (ulysses.py:39-40)."""


class ShapeError(ValueError):
    """Operand shapes are incompatible (tensor.py:23-24)."""


class DegenerateRowError(ValueError):
    """A softmax row has no unmasked entries (tensor.py:31-32)."""


class NativeError(RuntimeError):
    """CUDA runtime/driver failure inside the native library."""


# C-ABI status -> exception (include/ulysses_b200.h)
STATUS = {
    -1: DivisibilityError,
    -2: GroupDesyncError,
    -3: KernelError,
    -4: ForwardStateError,
    -5: ShapeError,
    -6: DegenerateRowError,
    -7: NativeError,
    -8: ValueError,
}
