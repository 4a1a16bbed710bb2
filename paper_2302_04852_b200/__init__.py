"""B200-native SparseProp hot path (arXiv 2302.04852).

Forward and backward of linear and 2-D conv layers whose weights carry a
fixed unstructured sparsity mask, as hand-written sm_100a CUDA kernels behind
the C ABI in include/sparseprop.h (libsparseprop.so, built in-tree).

    from paper_2302_04852_b200 import sparseprop as sp
    W = sp.sp_weight_create(dense_cuda, mask_cuda)
    Y = sp.sp_linear_fwd(W, X)            # X [C x B] -> Y [R x B]

`nn` holds drop-in `SparseLinear` / `SparseConv2d` modules with the paper's
§4.2 dense/sparse dispatcher; `dp` the data-parallel sparse MLP step (north
star cfg5); `prune` magnitude pruning and the GMP schedule (mask updates).
"""
__all__ = ["sparseprop", "nn", "dp", "prune"]
