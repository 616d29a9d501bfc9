"""B200-native fleet-placement hot path (arXiv 2001.05291, reference `fleetplace`).

Public API: paper_2001_05291_b200.fleetplace mirrors the reference's solver
interface; the C ABI is include/fleetplace_b200.h.
"""
