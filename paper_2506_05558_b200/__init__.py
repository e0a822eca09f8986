"""B200-native mini bundle adjustment: sm_100a kernels (csrc/), their C ABI
(include/miniba.h), the ctypes binding and the batched host driver."""
from . import synth  # noqa: F401
