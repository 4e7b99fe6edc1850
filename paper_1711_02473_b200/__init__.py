"""B200-native (sm_100a) sum-factorised finite-element cell kernels.

Drop-in for the hot path of the reference ``sumfact`` package (arXiv
1711.02473, FInAT + TSFC): plan construction keeps the reference's Python
names (``compile_kernel``, ``REGISTRY``, ``action_form``, element and
quadrature builders) and the per-cell ABI metadata of its ``LoopProgram``;
batched cell-wise evaluation (``evaluate_batched``) runs hand-written fp64
CUDA kernels through the C-ABI library ``libsfk.so`` (``include/sfk.h``).
"""

from .errors import (ArityMismatch, DimensionMismatch, ExtentMismatch,
                     InvalidArity, InvalidDegree, NativeError, ShapeMismatch,
                     UnboundVariable, Unsupported, UnsupportedCell, UsageError)
from .quadrature import (gauss_legendre, gauss_lobatto_legendre,
                         gauss_legendre_points, gauss_lobatto_legendre_points,
                         tensor_rule)
from .elements import (coordinate_element, lagrange_interval, lagrange_tables,
                       scalar_element, tensor_product_element, vector_element)
from .forms import (REGISTRY, FormSpec, action_form, default_quadrature,
                    form_element, neohookean_residual_form)
from .plan import KernelPlan, compile_form, compile_kernel
from .loopprogram import LoopProgramPlan, load_program, program_flops
from .runtime import (evaluate_batched, evaluate_batched_pair, evaluate_host,
                      launch_count, load_library, sum_squares)

__version__ = "0.1.0"
