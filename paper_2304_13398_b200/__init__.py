"""B200-native 4-value timing-aware gate-level re-simulation (arxiv 2304.13398 hot path).

The compute path is the C-ABI library libgls.so (include/gls.h); `gls` is its
thin Python binding.  `workloads` draws seeded synthetic inputs.
"""
