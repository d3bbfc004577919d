"""B200-native (sm_100a) implementation of the Flern hot path (arXiv 2311.02781).

The product is the C-ABI library lib/libflern.so (include/flern.h); `flern` is its thin
ctypes binding and `session` wires a datagen-style query configuration onto it.
"""
