"""Runtime knobs of the drop-in, mirroring the reference's ``annkit.config``
(config.py:1-12).

``blas_threshold``: query batches at or above this size use the matrix
decomposition path (the fused tcgen05 GEMM + top-k kernel, flat_search_blas
semantics, flat.py:94-118); smaller batches take the direct per-pair path
(flat_search, flat.py:76-91), as ``FlatIndex._search`` dispatches at
flat.py:58-62.  Read at every search.
"""

blas_threshold: int = 20
