"""Drop-in installation behind an unmodified ``blockten``.

The reference binds names at import time (``from .decomp import hosvd`` in
apps.py:26, ``from .blocks import struct_expand`` in reconstruct.py:25, the
long import lists of cli.py:22-60, ...), so replacing
``blockten.decomp.hosvd`` alone would leave every consumer on the CPU path.
``install()`` therefore rebinds each hot-path name in EVERY ``blockten``
module namespace that holds it -- functions, the result dataclasses (so the
reference's own ``isinstance`` checks in consumers see bt200's types) and the
exception classes (so ``except ShapeError`` in cli.py:383-397 catches bt200's
errors).  ``uninstall()`` restores the saved bindings.

The seeded-init hook stays the reference's: decomp.py:372 resolves the
module-level ``_cp_init`` at call time, and users override
``blockten.decomp._cp_init``.  While installed, bt200's ``cp_als`` calls that
hook when a user has replaced it and bt200's device HOSVD init otherwise.

Nothing here computes; the rebound names are the package's public API.
"""

from __future__ import annotations

import importlib
import sys

import pkgutil


def _modules(package: str) -> list:
    """The package and every module in it (blockten/__init__.py:12-89
    re-exports the hot-path names; each other module -- fileio, cli, ... --
    imports what it uses at module level, errors included), so no consumer
    keeps a reference binding."""
    pkg = importlib.import_module(package)
    names = [package]
    for info in pkgutil.iter_modules(getattr(pkg, "__path__", [])):
        if not info.name.startswith("__"):
            names.append(f"{package}.{info.name}")
    return names

# name -> "module.attr" inside this package
_TARGETS = {
    # tensor.py
    "unfold": "tensor.unfold", "fold": "tensor.fold", "mode_multiply": "tensor.mode_multiply",
    "fro_norm": "tensor.fro_norm", "twist": "tensor.twist", "squeeze": "tensor.squeeze",
    # blocks.py
    "BlockPattern": "blocks.BlockPattern", "build_pattern": "blocks.build_pattern",
    "classify_placements": "blocks.classify_placements", "detect_pattern": "blocks.detect_pattern",
    "extract_blocks": "blocks.extract_blocks", "mat_to_tensor": "blocks.mat_to_tensor",
    "tensor_to_mat": "blocks.tensor_to_mat", "struct_expand": "blocks.struct_expand",
    "struct_scalars": "blocks.struct_scalars", "struct_assemble": "blocks.struct_assemble",
    # decomp.py
    "TuckerRep": "decomp.TuckerRep", "KruskalRep": "decomp.KruskalRep",
    "CpResult": "decomp.CpResult", "svd_truncated": "decomp.svd_truncated",
    "qr_thin": "decomp.qr_thin", "cholesky": "decomp.cholesky", "_mode_basis": "decomp._mode_basis",
    "hosvd": "decomp.hosvd", "tucker_partial": "decomp.tucker_partial", "cp_als": "decomp.cp_als",
    # reconstruct.py
    "FlopCounter": "reconstruct.FlopCounter", "KronSumRep": "reconstruct.KronSumRep",
    "BlockLowRankRep": "reconstruct.BlockLowRankRep",
    "TuckerBlockRep": "reconstruct.TuckerBlockRep",
    "kron_sum_from_tucker": "reconstruct.kron_sum_from_tucker",
    "kron_sum_from_kruskal": "reconstruct.kron_sum_from_kruskal",
    "blr_from_tucker": "reconstruct.blr_from_tucker",
    "blr_from_kruskal": "reconstruct.blr_from_kruskal", "matvec": "reconstruct.matvec",
    "densify": "reconstruct.densify", "error_fro": "reconstruct.error_fro",
    # psd.py
    "SpsdRep": "psd.SpsdRep", "SpdRep": "psd.SpdRep",
    "check_transpose_closed": "psd.check_transpose_closed",
    "spsd_compress_blocks": "psd.spsd_compress_blocks", "spsd_compress": "psd.spsd_compress",
    "spd_compress": "psd.spd_compress",
    # multilevel.py
    "MultilevelPattern": "multilevel.MultilevelPattern",
    "MultilevelTuckerRep": "multilevel.MultilevelTuckerRep", "MlKronTerm": "multilevel.MlKronTerm",
    "psf_weighted_tensor": "multilevel.psf_weighted_tensor",
    "ml_kron_sum_from_tucker": "multilevel.ml_kron_sum_from_tucker",
    # apps.py
    "MarkovSequence": "apps.MarkovSequence", "LtiSystem": "apps.LtiSystem",
    "EraResult": "apps.EraResult", "markov_from_lti": "apps.markov_from_lti",
    "hankel_pattern_from_markov": "apps.hankel_pattern_from_markov",
    "era_identify_compressed": "apps.era_identify_compressed",
    # container.py
    "container_write": "container.container_write", "container_read": "container.container_read",
    "container_kind": "container.container_kind",
    # errors.py (errors.py:11-32)
    "ShapeError": "errors.ShapeError", "PatternMismatchError": "errors.PatternMismatchError",
    "NotPositiveDefiniteError": "errors.NotPositiveDefiniteError",
    "ConvergenceError": "errors.ConvergenceError",
    "ContainerFormatError": "errors.ContainerFormatError",
    "ContainerExtentError": "errors.ContainerExtentError",
}

_saved: dict = {}          # (module name, attr) -> original object
_state: dict = {}


def _resolve(path: str):
    mod, attr = path.split(".")
    return getattr(importlib.import_module(f"{__package__}.{mod}"), attr)


def install(package: str = "blockten") -> dict:
    """Route ``package`` (default: the reference ``blockten``) through bt200.

    Imports every module of the package (a module that fails to import,
    e.g. cli, is skipped) and rebinds each name of ``_TARGETS`` it holds.
    Returns ``{module: [rebound names]}``.  Idempotent; ``uninstall()``
    reverts.  Raises ImportError when the package itself is absent."""
    from . import decomp as bdecomp

    importlib.import_module(package)
    if _state.get("package") not in (None, package):
        uninstall()
    done: dict = {}
    for modname in _modules(package):
        try:
            mod = importlib.import_module(modname)
        except ImportError:
            continue
        hits = []
        for attr, path in _TARGETS.items():
            if attr in vars(mod):
                key = (modname, attr)
                if key not in _saved:
                    _saved[key] = vars(mod)[attr]
                setattr(mod, attr, _resolve(path))
                hits.append(attr)
        done[modname] = hits
    # seeded-init hook: keep the reference's decomp._cp_init the one users set
    if "bt_cp_init" not in _state:
        ref_decomp = sys.modules.get(package + ".decomp")
        bt_default = bdecomp._cp_init
        _state["bt_cp_init"] = bt_default

        def _is_ref_default(hook) -> bool:
            # the reference's own HOSVD init (decomp.py:329-341), recognised by
            # where it is defined -- a hook the user set before install() is
            # honoured like one set after it
            return (getattr(hook, "__module__", None) == ref_decomp.__name__
                    and getattr(hook, "__qualname__", None) == "_cp_init")

        def _cp_init(t, r):
            hook = getattr(ref_decomp, "_cp_init", None)
            if hook is not None and not _is_ref_default(hook):
                return hook(t, r)
            return bt_default(t, r)

        bdecomp._cp_init = _cp_init
    _state["package"] = package
    return done


def uninstall() -> None:
    """Restore every binding ``install()`` replaced."""
    from . import decomp as bdecomp

    for (modname, attr), obj in list(_saved.items()):
        mod = sys.modules.get(modname)
        if mod is not None:
            setattr(mod, attr, obj)
    _saved.clear()
    if "bt_cp_init" in _state:
        bdecomp._cp_init = _state.pop("bt_cp_init")
    _state.pop("package", None)


def installed() -> bool:
    return "package" in _state
