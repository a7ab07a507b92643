"""B200-native (sm_100a) sparse triangular solve -- arXiv 1710.04985's hot path.

* ``sptrsv``    -- ctypes binding of include/sptrsv.h (libsptrsv.so, built in-tree);
                   import it explicitly: ``from paper_1710_04985_b200 import sptrsv``
* ``partition`` -- batch partitioner for independent RHS across ranks
* ``build``     -- nvcc build of the library
"""
from . import partition  # noqa: F401
