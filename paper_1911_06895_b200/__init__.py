"""B200-native drop-in for the reference's delta-stepping SSSP path."""
from .containers import (  # noqa: F401
    SparseMatrix, SparseVector, mask_from_indices, matrix_build, vector_build,
)
