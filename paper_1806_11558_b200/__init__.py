"""B200-native (sm_100a) hot path of Harbrecht & Zaspel, arXiv 1806.11558: H-matrix BEM
(tree build, batched ACA, batched near-field assembly, batched H-matvec, CG/GMRES, multi-GPU
leaf partition) behind the C ABI of include/hm.h.  See DESIGN.md."""
from .hm import HMatrix, HMError, lib  # noqa: F401
