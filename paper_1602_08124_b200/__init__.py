"""B200-native vDNN (arXiv 1602.08124): bit-exact planner + CUDA executor.

Python mirror of the reference's network-definition and offload-policy API
(vdnnsim). See include/vdnn.h for the C ABI and DESIGN.md for the design.
"""
