"""B200-native block eigensolver (arXiv 2409.05572 hot path).

The product is ``libblockeig_b200.so`` (hand-written sm_100a kernels behind the
reference's ``blockeig.h`` C interface).  ``load()`` binds it with ctypes; there
is no CPU fallback: loading fails loudly when the library was not built.
"""
import os

from . import blockeig  # noqa: F401

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libblockeig_b200.so")


def load():
    """Bind the B200 library (raises if it has not been built)."""
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() first")
    return blockeig.Library(LIB_PATH)
