"""Drop this package's GPU AxLocal into the reference package (``hosfem``).

The reference exposes AxLocal as a Python class API, not a plugin registry
(SURVEY §8(b)): ``hosfem.axlocal.LocalOperator``, ``ax_local_apply`` and
``dense_local_matrix`` (reference axlocal.py:115-310), imported by name into
``hosfem.solver``, ``hosfem.verify`` and ``hosfem.cli``.  ``patch_hosfem``
rebinds those names in every loaded ``hosfem`` module to this package's
implementations, which accept the reference's own objects unchanged (its
KernelSpec and enums, Element list, SpectralBasis, LocalField, coefficient
fields) and return LocalFields with ``.data``.  After the patch the
reference's solver, verification and tests run on the B200 kernels; there is
no CPU fallback behind it.

    import hosfem, paper_2504_07042_b200.compat as compat
    restore = compat.patch_hosfem(hosfem)
    ...                      # hosfem.LocalOperator is now the GPU operator
    restore()

This is the binding INTEGRATION.md §1 describes; tests/test_reference_suite_gpu.py
runs the reference's own operator tests through it.
"""

from __future__ import annotations

import sys

from . import axlocal

#: the reference entry points this package replaces, by name
ENTRY_POINTS = ("LocalOperator", "ax_local_apply", "dense_local_matrix")


def patch_hosfem(hosfem=None):
    """Rebind the reference's AxLocal entry points to this package's; returns a
    ``restore()`` callable that puts the originals back."""
    if hosfem is None:
        import hosfem  # noqa: F811 - the caller's reference installation
    originals = {name: getattr(hosfem.axlocal, name) for name in ENTRY_POINTS}
    replaced = []
    prefix = hosfem.__name__
    for modname, mod in list(sys.modules.items()):
        if mod is None or not (modname == prefix or modname.startswith(prefix + ".")):
            continue
        for name, orig in originals.items():
            if getattr(mod, name, None) is orig:
                setattr(mod, name, getattr(axlocal, name))
                replaced.append((mod, name, orig))

    def restore():
        for mod, name, orig in replaced:
            setattr(mod, name, orig)

    return restore
