"""B200-native Interpretable-Generalization intersect-and-subset search.

The compute lives in libig_b200.so (hand-written sm_100a kernels behind the
C-ABI in include/ig_b200.h); this package is the Python mirror of the
reference's KernelBackend / mine / pipeline interface over that ABI.  Importing
the package does not load the native library; importing ``api`` does, and fails
loudly when it is not built.
"""

__all__ = ["api", "synth"]
