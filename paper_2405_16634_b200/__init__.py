"""paper_2405_16634_b200 — B200-native (sm_100a) WNNC hot path (arXiv 2405.16634).

The compute path lives in ``libwn.so`` (hand-written CUDA behind the C ABI of ``include/wn.h``);
``paper_2405_16634_b200.wn`` is the thin ctypes binding.  Importing the package itself has no side
effects so that ``synth`` (seeded input generators) can be used without a GPU.
"""
