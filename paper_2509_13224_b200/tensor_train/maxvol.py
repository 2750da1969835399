"""maxvol on the device (reference tensor_train/maxvol.py): cooperative GEPP row choice + greedy
Sherman-Morrison swaps with lowest-index tie-break, one kernel launch."""

from ..linalg import MaxvolError, maxvol, maxvol_colmajor

__all__ = ["MaxvolError", "maxvol", "maxvol_colmajor"]
