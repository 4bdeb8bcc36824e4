"""B200-native light-field Richardson-Lucy hot path of AutoDeconJ (arXiv 2208.11422).

The product is the C-ABI library ``liblfm.so`` (include/lfm.h) built from ``csrc/`` for sm_100a;
``lfm`` is its thin ctypes binding.  There is no CPU fallback: touching any binding attribute loads
``liblfm.so`` and raises ImportError if it is missing.  (``build`` is importable without the library.)
"""
_EXPORTS = ("LfmError", "Plan", "lfm_comm_unique_id", "lfm_dct_entropy", "lfm_plan_estimate", "lfm_policy_default",
            "lfm_version", "make_optics", "make_policy")


def __getattr__(name):
    if name in _EXPORTS:
        from . import lfm
        return getattr(lfm, name)
    raise AttributeError(name)
