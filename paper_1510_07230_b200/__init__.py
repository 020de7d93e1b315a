"""B200-native hot path of arXiv 1510.07230 (parallel orbital-updating
Kohn-Sham energy minimisation): sm_100a kernels behind the C ABI in
include/parorb_gpu.h, a C++ mirror of the reference solver loop, and a thin
Python binding (`paper_1510_07230_b200.native`). See DESIGN.md."""
from . import configs, rng  # noqa: F401
