"""scalarmc_b200 — B200-native particle forward map G(u) of arXiv 1808.10580.

Drop-in for the hot path of the reference library scalarmc: observe_ad /
observe_ad_single / observe_bvp (and the u -> G callers misfit / forcing_cost)
run as fused sm_100a kernels behind the C ABI in include/scalarmc_b200.h.
"""
from .api import (  # noqa: F401
    AdObservation,
    AdProblemSpec,
    Bump,
    ChainConfig,
    BvpProblemSpec,
    Context,
    CosineTerm,
    DiffusionModel,
    Domain,
    ESTIMATE_DTYPE,
    ForcingBasis,
    ForcingControl,
    FourierVelocityField,
    LikelihoodSpec,
    NelderMeadOptions,
    ParticleEstimate,
    Point2,
    Precision,
    PriorSpec,
    ScalarField,
    StepScheme,
    Vec2,
    VelocityField,
    VelocityMode,
    ad_particle_values,
    bvp_particle_values,
    default_context,
    nccl_unique_id,
    forcing_basis,
    GalerkinBasis,
    GalerkinResult,
    galerkin_field_grid,
    galerkin_solve_ad,
    galerkin_spectral_radius,
    forcing_cost,
    nelder_mead,
    optimize_forcing,
    normal_pairs_device,
    observe_ad,
    observe_ad_batched,
    observe_ad_single,
    observe_bvp,
    observe_bvp_range,
    philox_device,
    prior_draw,
    run_chains,
    velocity_from_coefficients,
)
from ._abi import LIB_PATH, load_library  # noqa: F401

__version__ = "0.1.0"
