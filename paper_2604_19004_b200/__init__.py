"""B200-native estimation-based SpGEMM (placeholder during bring-up)."""
from .csr import CsrMatrix, from_triplets, identity, transpose, validate  # noqa: F401
