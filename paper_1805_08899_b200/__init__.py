"""paper_1805_08899_b200 — B200-native (sm_100a) hot path of Echo (arXiv 1805.08899).

    abi.py      ctypes binding of libecho.so (include/echo.h); marshalling only
    build.py    nvcc build of csrc/ into libecho.so (sm_100a)
    nmt.py      NMT training step around the ABI (STASH / RECOMPUTE), cuBLAS FCs outside the hot path
    dp.py       batch-sharded data parallelism (NCCL allreduce of flat fp32 gradients)
    graphs.py   graph documents for the footprint estimator, mirroring the GPU path's op structure

There is no CPU fallback: without libecho.so or a CUDA device the ops raise.
"""
__all__ = ["abi", "build"]
