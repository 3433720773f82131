"""B200-native split-step Fourier propagator for the 3D TDSE on the CTAP
atom-chip grid (arXiv:1309.2451), a drop-in for the hot path of the
reference package `ctapsim`: make_plan -> evolve_real -> _advance, with the
potential kernel and the observer reductions.

Python here is the host-side mirror of the reference interface; the compute
is hand-written CUDA for sm_100a in libctap.so (csrc/, C ABI in
include/ctap.h).  Modules mirror the reference module names:

    qgrid        SimGrid, make_grid, Wavefunction (HBM-resident), gaussian_packet, QWF1 I/O
    propagator   make_plan, step, evolve_real, energies, ground_state_imaginary, observers
    observables  populations, edge_density, density_xz, PopulationRecorder, EdgeMonitor
    magfield     ChipSegments, assemble_potential (bit-exact device Biot-Savart)
    slab         x-slab decomposition over torch.distributed (NCCL all-to-all)
"""

__version__ = "0.1.0"

from . import constants, magfield, observables, propagator, qgrid  # noqa: F401
from ._lib import LIB_PATH, load as load_library  # noqa: F401
