"""B200-native fine stages of Multistage SfM (arXiv 1512.06235).

Drop-in replacements for the reference package's hot-path entry points
(msfm.guided.guided_match_pair, ...), backed by hand-written sm_100a CUDA
kernels in libmsfm_b200.so.  No CPU fallback exists: without the library or
a CUDA device the entry points raise DeviceUnavailableError.
"""

__version__ = "0.1.0"
