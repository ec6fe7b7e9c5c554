"""B200-native fine stages of Multistage SfM (arXiv 1512.06235).

Drop-in replacements for the reference package's hot-path entry points
(msfm.guided.guided_match_pair, ...), backed by hand-written sm_100a CUDA
kernels in libmsfm_b200.so.  No CPU fallback exists: without the library or
a CUDA device the entry points raise DeviceUnavailableError.
"""

__version__ = "0.1.0"

# use the caller's msfm classes (errors, Match, FeatureRef, ...) when the
# reference package is importable (types.adopt_reference_types)
from .types import adopt_reference_types as _adopt

_adopt()


def reserve_device_memory(gigabytes: float, device=None) -> None:
    """Grow PyTorch's caching allocator by one block of ``gigabytes`` and release it
    to the cache: later stage buffers are carved from it instead of each paying a
    fresh ``cudaMalloc`` (tens of ms apiece on a fresh process), which is what makes
    a pipeline's first call of every stage slow."""
    import torch

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if isinstance(device, int):
        dev = torch.device("cuda", device)
    # PyTorch caches the freed block for the stream it was allocated on: only later
    # allocations on the current stream of `dev` are carved from it
    with torch.cuda.device(dev):
        block = torch.empty(int(gigabytes * (1 << 30)), dtype=torch.uint8, device=dev)
        del block
