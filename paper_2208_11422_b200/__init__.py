"""B200-native light-field Richardson-Lucy hot path of AutoDeconJ (arXiv 2208.11422).

The product is the C-ABI library ``liblfm.so`` (include/lfm.h) built from ``csrc/`` for sm_100a;
``lfm`` is its thin ctypes binding.  There is no CPU fallback.
"""
from .lfm import (LfmError, Plan, lfm_comm_unique_id, lfm_dct_entropy, lfm_plan_estimate, lfm_policy_default,  # noqa: F401
                  lfm_version, make_optics, make_policy)
