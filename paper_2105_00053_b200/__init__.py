"""B200-native posit-quire kernels (arxiv 2105.00053 hot path).

The exact quire-accumulated posit dot product behind Conv2d / Linear
(forward, input-gradient and weight-gradient passes), hand-written for
sm_100a and exposed through the C-ABI in include/pnn_b200.h.
"""
from .ops import P80, P81, P82, P121, P161, PositConfig, matmul, par_matmul, quire_gemm  # noqa: F401

__all__ = ["PositConfig", "P80", "P81", "P82", "P121", "P161", "matmul", "par_matmul", "quire_gemm"]
