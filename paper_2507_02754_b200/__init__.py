"""B200-native sliding-window 2-simplicial attention (arXiv 2507.02754).

The compute lives in ``libsimplicial.so`` (hand-written sm_100a CUDA behind the C ABI in
``include/simplicial_attn.h``); ``binding`` is a thin ctypes layer with the same names.
PyTorch only provides device memory, streams and process groups.  There is no CPU
fallback: every entry point raises if the CUDA library or a CUDA device is missing.
"""
from .binding import (  # noqa: F401
    SA_FORCE_SIMT, SA_IN_F32, SA_OUT_F32, SA_VARIANT_DET, SA_PATH_SIMT, SA_PATH_TCGEN05,
    backward, bwd_path, forward, fwd_path, host_step, launch_count, lib, load_library,
    profile_enable, profile_read,
)
from .autograd import SimplicialAttnFunction, simplicial_attention  # noqa: F401,E402
