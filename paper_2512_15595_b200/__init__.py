"""B200-native bulk Bloom filters (arXiv 2512.15595): bulk add / contains over
blocked, register-blocked, sectorized and cache-sectorized filters.

* ``paper_2512_15595_b200.bf``     -- ctypes binding of libbf200.so (include/bf.h);
                                      importing it without the built library raises
* ``paper_2512_15595_b200.layout`` -- host-side Θ/Φ layout algebra
* ``paper_2512_15595_b200.dist``   -- multi-GPU build / lookup over torch.distributed
* ``paper_2512_15595_b200.build``  -- nvcc build of the library for sm_100a
"""
__all__ = ["bf", "layout", "dist", "build"]
