"""B200-native level-batched recursive skeletonization (arXiv 2001.11619).

Drop-in for the hot path of the reference package ``skelsolve``
(``__init__.py:9-19``): ``factor``, ``update``, ``Factorization.solve`` /
``apply`` with the same signatures and observables, computed by the sm_100a
kernels of ``libskelb200.so``.
"""

from .geometry import (AddHole, Boundary, Curve, DeleteHole, GeometryError, MoveHole,
                       PerturbationReport, apply_perturbation)
from .tree import Tree, TreeError, build_tree, default_root_box, proxy_radius, refit_tree
from .skel import (BoxFactors, Factorization, LAPLACE, RootBoxExceededError, SingularPivotError, STOKES,
                   SystemSpec, evaluate_interior, factor, point_in_domain,
                   system_matvec, update)

__version__ = "0.1.0"
