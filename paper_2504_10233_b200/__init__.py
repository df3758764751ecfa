"""B200-native hot path of Bingo (arXiv 2504.10233): radix-factorised sampling
structures, batched walker step and batched updates, behind the C-ABI of
include/bingo.h (libbingo.so).  See DESIGN.md."""
from .bingo import (DEEPWALK, NODE2VEC, PPR, EMPTY, ONE, DENSE, SPARSE, REGULAR, NO_CAP, BingoError,  # noqa: F401
                    Graph, ABI_SYMBOLS, LIB_PATH)
