"""B200-native snapshot engine (DataStates-LLM lazy capture path, arXiv 2601.16956).

The product is ``_lib/libts_b200.so`` (C-ABI in ``include/ts_b200.h``: host C++
runtime + sm_100a kernels). ``api`` mirrors the reference's State Provider API
in Python on top of it (``from paper_2601_16956_b200 import api``);
``synthetic`` builds the configs of BASELINE.json.
"""
from . import synthetic  # noqa: F401  (pure Python, no CUDA needed)
