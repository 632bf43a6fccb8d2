"""B200-native gamma-EigenGame (arxiv 2206.04993): the data-parallel hot path
of Alg. 2 (minibatch products, k x k Gram tables, penalty sums, fused
ascent / retraction / auxiliary update) as hand-written sm_100a CUDA behind
the C ABI in include/geig.h.  `geig` is the ctypes binding; `parallel` holds
the multi-GPU host logic (row sharding + all-reduce of the products)."""
