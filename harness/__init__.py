"""Benchmark / test harness (not the product): the synthetic scene generator
that builds the same float32 pairs as the reference's `hdrflow.synth` on a
box where /root/reference does not exist."""
