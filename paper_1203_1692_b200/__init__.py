"""B200-native SpAMM multiply path (arXiv 1203.1692).

Drop-in for the multiply path of the reference package ``spamm``
(`pkg/src/spamm/__init__.py:10-59` re-exports the same names): build operands with
``QuadtreeMatrix.from_dense``, then ``multiply(a, b, MultiplyConfig(tau=...))``.
All arithmetic runs in hand-written CUDA kernels for sm_100a behind the C ABI in
``include/spamm_b200.h``; there is no CPU or PyTorch fallback.
"""

from .morton import c_index, decode, encode, k_match, k_of_a, k_of_b  # noqa: F401
from .tree import DEFAULT_BLOCK, DenseMatrix, QuadtreeMatrix, TreeNode, drop_tolerance, tree_depth  # noqa: F401
from .io import QUADTREE_MAGIC, MatrixFormatError, load_quadtree, save_quadtree  # noqa: F401
from .symbolic import MultiplyPlan, PlanStats, ProductTask, build_plan, plan_dump, plan_stats  # noqa: F401
from .numeric import (  # noqa: F401
    GRANULARITIES,
    MICRO_FLOPS,
    ExecCounters,
    MultiplyConfig,
    execute_plan,
    multiply,
)
from .hosttree import HostTree, multiply_host, multiply_host_parts  # noqa: F401

__version__ = "0.1.0"
