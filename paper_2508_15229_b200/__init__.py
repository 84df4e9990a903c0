"""B200-native tailored LM-head path of VocabTailor (arXiv 2508.15229).

The compute lives in ``lib/libsvt.so`` (hand-written sm_100a CUDA behind the
C-ABI in ``include/svt.h``); the C++ drop-in of the reference API is
``lib/libsubvocab_b200.so`` (``include/subvocab/*.hpp``). This package is the
Python host mirror used by tests and ``bench.py``. Importing the compute
modules fails loudly when the CUDA library has not been built.
"""
__version__ = "0.1.0"
