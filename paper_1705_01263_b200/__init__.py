"""paper_1705_01263_b200 -- B200-native light-transport hot path of the Iray paper (arXiv 1705.01263).

Drop-in for the reference package `lumenwave`'s kernel module and render entry:
  core.kernels   halton_batch / intersect_batch / oct / pixel filter on sm_100a
  qmc            DimensionTable and exact QMC helpers (host tables)
  geometry       flatten_instances, GPU build_bvh, intersect wrappers
  render         Renderer / render(): wavefront or megakernel path tracing, NEE + MIS
  distributed    sample-space partition + NCCL framebuffer reduction
"""

__version__ = "0.1.0"
