"""paper_2302_06126_b200 — B200-native SFB gradient synchronisation (TAG, arXiv 2302.06126).

Submodules (imported explicitly, nothing is loaded eagerly):
  tag    ctypes binding of libtag.so (the C ABI declared in include/tag.h); argument marshalling only
  synth  seeded synthetic inputs shaped like the paper's workloads (no method arithmetic)
  dist   torch.distributed plumbing: NCCL-id bootstrap, rank shards, max-over-ranks timing
"""
__version__ = "0.1.0"
