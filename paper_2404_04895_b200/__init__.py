"""TensorACO-B200: the TensorACO hot path (one ACO iteration with IR / AdaIR
selection) as hand-written sm_100a CUDA behind the reference package's Python
API (``antbatch``, arXiv 2404.04895).

Drop-in names (same signatures and exceptions as the reference):
    compute_probability_matrix, construct_tours, init_starts, batch_costs,
    tour_cost, select_elite, accumulate_increments, apply_update,
    edge_index_matrix, increment_matrix, gamma_at, scaled_log_weights,
    AcoParams, GammaSchedule, PheromoneState, ProbabilityMatrix, TourBatch,
    TspInstance, Selection, euclidean_instance, NumericalUnderflow, ...
plus the device-resident ``Solver(instance, params).step() / .run()``.
Importing is CPU-safe; every compute call needs a CUDA device and the
in-tree libtaco.so (no CPU fallback).
"""

from .colony import (
    NumericalUnderflow,
    batch_costs,
    compute_probability_matrix,
    construct_tours,
    init_starts,
    tour_cost,
)
from .model import (
    TAU_MIN,
    AcoParams,
    DegenerateInstance,
    GammaSchedule,
    InvalidPermutation,
    PheromoneState,
    ProbabilityMatrix,
    Selection,
    TourBatch,
    TspInstance,
    euclidean_instance,
    instance_from_distances,
)
from .pheromone import (
    accumulate_increments,
    apply_update,
    edge_index_matrix,
    increment_matrix,
    select_elite,
)
from .selection import AllZeroWeights, argmax_select_block, gamma_at, scaled_log_weights
from .solver import Solver
from ._device import DeviceInstance, UnsupportedEdgeWeightType, device_build_instance

device_euclidean_instance = DeviceInstance.from_coords

__version__ = "0.1.0"

__all__ = [
    "AcoParams", "AllZeroWeights", "DegenerateInstance", "GammaSchedule", "InvalidPermutation",
    "NumericalUnderflow", "PheromoneState", "ProbabilityMatrix", "Selection", "Solver", "TAU_MIN",
    "TourBatch", "TspInstance", "accumulate_increments", "apply_update", "batch_costs",
    "compute_probability_matrix", "construct_tours", "edge_index_matrix", "euclidean_instance",
    "gamma_at", "argmax_select_block", "increment_matrix", "init_starts", "instance_from_distances", "scaled_log_weights",
    "select_elite", "tour_cost", "DeviceInstance", "device_euclidean_instance",
    "device_build_instance", "UnsupportedEdgeWeightType",
]
