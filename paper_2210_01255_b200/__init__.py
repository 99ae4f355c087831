"""B200-native Spectral Ewald engine (stokeslet / stresslet / rotlet, D = 0..3).

Drop-in for the reference host API (select_parameters, full_potential,
se_fourier_potential, realspace_potential, spread, gather and the stage
functions aft_forward, scale, aft_inverse, precompute_0p); the numeric work
runs in sm_100a CUDA kernels behind the C-ABI of include/sewald_gpu.h.
"""
from .api import (Cell, DeviceError, DomainError, Engine, EstimateReport, EwaldParams, GridSpec,
                  InvalidArgument, Kernel, ParameterSelection, SePipelineOptions, SelectionOptions,
                  Session, SewaldError, SewaldRuntimeError, SourceSystem, TargetSet, ToleranceSpec,
                  UpsamplingPlan, WindowKind, WindowSpec, build_grid, default_engine, full_potential,
                  gather, pkb_coefficients, realspace_potential, se_fourier_potential,
                  select_parameters, source_quantity, spread, strength_components, window_eval,
                  window_hat, ModifiedKernelSpec, FourierField, PrecomputedKernel0P, aft_forward,
                  aft_inverse, scale, precompute_0p, KernelOption, get_kernel_option,
                  set_kernel_option, kernel_options, MultiEngine)

__all__ = [n for n in dir() if not n.startswith("_")]
from . import analytic  # noqa: E402,F401  (GPU analytic oracles, SPEC module 'reference')
