"""B200-native (sm_100a) graph-partitioned MLIP inference path (DistMLIP -> graphmd).

The compute lives in libgraphmd_b200.so (C ABI: include/graphmd_b200.h); this
package is the Python mirror of the reference's plugin API over that ABI.
"""
from .graphmd import (  # noqa: F401
    AtomGraph, AtomicSystem, AtomPartition, BondSet, Buckets, Distributed, DistributedFeatures,
    Error, LineGraphPartition, PartitionedAtomGraph, PartitionedLineGraph, PartitionRule,
    PotentialOutput, SpanLayout, StepTiming, ToyPotentialParams, build_neighbor_list,
    forward_distributed, lib, make_supercell, random_perturb, rng_uniform,
)

__all__ = [n for n in dir() if not n.startswith("_")]
