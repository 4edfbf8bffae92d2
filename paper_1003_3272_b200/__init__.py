"""paper_1003_3272_b200 -- B200-native MM (majorize-minimize) iteration
kernels for Zhou, Lange & Suchard (arXiv 1003.3272), as a drop-in for the
reference package's solver API (mmkit 0.1.0, ``pkg/src/mmkit/__init__.py``).

Solvers: Frobenius NNMF (``nnmf_run``), penalized PET reconstruction
(``pet_run``) and stress-majorization MDS (``mds_run``), each with its
single-step and objective functions, ``MmConfig`` stopping rules and
``MmTrace`` objective traces.  All iteration arithmetic runs in hand-written
sm_100a CUDA (``libmmk.so``); there is no CPU fallback.
"""

from .backend import SERIAL, Backend
from .datasets import (PetGeometry, build_neighborhoods, build_system_matrix,
                       cbcl_preprocess, default_phantom, simulate_counts,
                       synthetic_votes, votes_to_dissimilarity)
from .driver import MmConfig, MmProblem, MmTrace, relative_change, run_mm
from .errors import (DeviceError, DomainError, InputError, MatrixFormatError, MmkitError,
                     MonotonicityError, NonFiniteError, NumericsError, ShapeError)
from .io import load_matrix_device, read_mmx_header
from .kernels import elementwise, matmul, matvec, tree_reduce_sum
from .mds import (MdsProblem, PackedMdsProblem, anchor_configuration, mds_run, mds_update, stress,
                  stress_gradient)
from .nnmf import (FactorPair, NnmfProblem, nnmf_gradient, nnmf_objective,
                   nnmf_poisson_objective, nnmf_poisson_run, nnmf_poisson_update, nnmf_run,
                   nnmf_surrogate, nnmf_update_v, nnmf_update_w)
from .pet import (PetProblem, SparsePetProblem, pet_loglik, system_matrix_device, pet_penalized_gradient, pet_penalized_objective,
                  pet_run, pet_surrogate, pet_update)

__version__ = "0.1.0"
