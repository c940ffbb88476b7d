"""B200-native CUDA backend for NMODL mechanisms (arXiv 1905.02241).

The reference compiler (`modlc`) keeps its front-end; this package supplies
the sm_100a code generator and the device runtime for its hot path,
nrn_state + nrn_cur over SoA instance data:

    emit_cuda(layout)            -> EmittedUnit("cuda", "<mech>.cu", text)
    CudaRunner(layout).run_kernel(data, kernel_name, steps)   # interp.Runner drop-in
    simulate(layout, data, steps)                             # interp.simulate drop-in

`layout` is a reference `MechanismLayout` or its JSON mirror `MechIR`.
"""

from .codegen_cuda import CudaOptions, EmittedUnit, UnsupportedConstruct, cuda_abi, emit_cuda
from .ir import MechIR, from_layout

__all__ = [
    "CudaOptions",
    "EmittedUnit",
    "MechIR",
    "UnsupportedConstruct",
    "cuda_abi",
    "emit_cuda",
    "from_layout",
    "CudaRunner",
    "InterpError",
    "simulate",
]


def __getattr__(name):
    # the runtime layer loads CUDA libraries; import it lazily
    if name in ("CudaRunner", "InterpError", "simulate", "DeviceInstanceData", "HostInstanceData"):
        from . import runner

        return getattr(runner, name)
    raise AttributeError(name)
