"""B200-native retrieval stage of RAGDoll (arXiv 2504.15302): batched IVF-Flat
search over a partly HBM-resident inverted-list index.

The product is the C-ABI library ``lib/librd_b200.so`` (CUDA for sm_100a +
C++ host code, header ``include/rd.h``); ``retriever`` is its ctypes binding.
"""
from .retriever import (ENGINE_PATH, Error, Index, InfeasibleError, Library, ParseError, SearchResult,
                        engine)

__all__ = ["ENGINE_PATH", "Error", "Index", "InfeasibleError", "Library", "ParseError", "SearchResult", "engine"]
