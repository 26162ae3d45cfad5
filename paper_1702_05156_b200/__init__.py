"""B200-native (sm_100a) grid-block Dual-Mode SGM motion masking (arXiv 1702.05156).

The hot path lives in libdmsgm.so behind the C ABI of include/dmsgm.h; the binding is
paper_1702_05156_b200.dmsgm.  The homography estimation that feeds it (include/dmsgm_klt.h)
is bound by paper_1702_05156_b200.klt.  See DESIGN.md.

The binding is imported lazily so that `python -m paper_1702_05156_b200.build` works on
a fresh checkout; touching any API name loads libdmsgm.so and raises ImportError when it
is missing (there is no CPU fallback).
"""
_API = ("Dmsgm", "DmsgmError", "Params", "dmsgm_params", "dmsgm_info", "dmsgm_buffers", "band_halo_needed", "prefilter", "warp_frames",
        "DMSGM_MC_MODELS", "DMSGM_MC_FRAME", "DMSGM_MASK_BYTES", "DMSGM_MASK_BITS",
        "DMSGM_IPC_BYTES", "lib", "load_library", "version",
        "EXPORTS", "DMSGM_OK", "DMSGM_EINVAL", "DMSGM_ENOMEM", "DMSGM_ECUDA", "DMSGM_ESTATE")

_KLT_API = ("Klt", "KltParams", "dmsgm_klt_params", "KLT_EXPORTS")   # include/dmsgm_klt.h (NEXT-4)

__all__ = list(_API) + list(_KLT_API)


def __getattr__(name):
    if name in _API:
        from . import dmsgm
        return getattr(dmsgm, name)
    if name in _KLT_API:
        from . import klt
        return getattr(klt, name)
    raise AttributeError(name)
