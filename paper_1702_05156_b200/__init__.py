"""B200-native (sm_100a) grid-block Dual-Mode SGM motion masking (arXiv 1702.05156).

The hot path lives in libdmsgm.so behind the C ABI of include/dmsgm.h; this
package is the thin Python binding.  See DESIGN.md.
"""
from .dmsgm import (DMSGM_ECUDA, DMSGM_EINVAL, DMSGM_ENOMEM, DMSGM_ESTATE, DMSGM_OK, EXPORTS,
                    Dmsgm, DmsgmError, Params, dmsgm_info, dmsgm_params, lib, load_library, version)

__all__ = ["Dmsgm", "DmsgmError", "Params", "dmsgm_params", "dmsgm_info", "lib", "load_library",
           "version", "EXPORTS", "DMSGM_OK", "DMSGM_EINVAL", "DMSGM_ENOMEM", "DMSGM_ECUDA",
           "DMSGM_ESTATE"]
