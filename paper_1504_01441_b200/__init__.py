"""B200-native drop-in for the `hdrflow` register+merge path (arXiv 1504.01441).

Submodules mirror the reference package one for one -- `pipeline`, `image`,
`matcher`, `weeding`, `geometry`, `densify`, `fusion`, `metering`, `fileio`,
`viz` -- and run on libhdrb200.so (hand-written sm_100a kernels behind
the C ABI in include/hdrb200.h). `runner.BatchRunner` is the many-pairs
throughput path, `dist` the pair sharding across GPUs. Importing the package
loads nothing; the CUDA library is opened on first use and there is no CPU
fallback. The synthetic scene generator used by the tests and the benchmark
lives outside the product, in `harness.synth`.
"""
