"""B200-native dense per-pixel stage of the real-time non-rigid mosaicking
pipeline (arXiv 2103.07414): node-field blending + mosaic update (K1/K2) and
the dense EMDQ field with per-pixel uncertainty (K3), as sm_100a CUDA kernels
behind the C ABI in include/nrm_b200.h.

The CUDA library is loaded lazily (``paper_2103_07414_b200.mosaic``) so the
package imports on machines without a GPU; every compute entry point fails
loudly when libnrm_b200.so is missing.
"""

__version__ = "0.1.0"
