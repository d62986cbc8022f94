"""install(): bt200 behind an unmodified `blockten`.

Binding-level checks (no compute, so they run on CPU): every consumer module
of the reference sees bt200's functions, result types and exception classes;
the seeded-init hook stays the reference's; uninstall() restores.  Skipped
where the reference package is not importable (the GPU box has no
/root/reference)."""
import dataclasses
import importlib
import inspect
import os
import sys

import pytest

REF = "/root/reference/pkg/src"
# the GPU box has no /root/reference: there the unmodified reference comes
# from its pip install under baseline/_ref (git-ignored, travels with the repo)
_BASE = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
for _p in (REF, _BASE):
    if os.path.isdir(os.path.join(_p, "blockten")) and _p not in sys.path:
        sys.path.append(_p)
        break
blockten = pytest.importorskip("blockten")

import paper_2105_01170_b200 as bt  # noqa: E402
from paper_2105_01170_b200 import dropin  # noqa: E402


@pytest.fixture
def installed():
    done = bt.install()
    try:
        yield done
    finally:
        bt.uninstall()


def test_rebinds_every_consumer(installed):
    import blockten.apps as apps
    import blockten.cli as cli
    import blockten.decomp as decomp
    import blockten.psd as psd
    import blockten.reconstruct as rec

    # apps.py:25-26, cli.py:22-60, psd.py:30-39, reconstruct.py:25-28, decomp.py
    assert apps.hosvd is bt.hosvd and apps.tucker_partial is bt.tucker_partial
    assert apps.struct_expand is bt.struct_expand and apps.build_pattern is bt.build_pattern
    assert cli.cp_als is bt.cp_als and cli.mat_to_tensor is bt.mat_to_tensor
    assert cli.matvec is bt.matvec and cli.mode_multiply is bt.mode_multiply
    assert psd._mode_basis is bt.decomp._mode_basis and psd.cholesky is bt.cholesky
    assert psd.extract_blocks is bt.extract_blocks and psd.unfold is bt.unfold
    assert rec.struct_scalars is bt.struct_scalars and rec.qr_thin is bt.qr_thin
    assert rec.fro_norm is bt.fro_norm
    assert decomp.cp_als is bt.cp_als and decomp.KruskalRep is bt.KruskalRep
    assert blockten.cp_als is bt.cp_als and blockten.matvec is bt.matvec
    # exception classes: `except ShapeError` in the CLI catches bt200's errors
    assert cli.ShapeError is bt.ShapeError and blockten.errors.ShapeError is bt.ShapeError
    assert installed["blockten.cli"] and installed["blockten.apps"]


def test_signatures_and_fields_match_reference():
    """Every rebound function takes the reference's parameters (in order; bt200
    may add keyword-only extensions) and every dataclass has its fields."""
    for attr, path in dropin._TARGETS.items():
        mods = [m for m in dropin._modules("blockten") if attr in vars(importlib.import_module(m))]
        if not mods:
            continue
        ref = vars(importlib.import_module(mods[0]))[attr]
        new = dropin._resolve(path)
        if dataclasses.is_dataclass(ref):
            assert [f.name for f in dataclasses.fields(ref)] == \
                [f.name for f in dataclasses.fields(new)], attr
        elif inspect.isfunction(ref):
            rp = list(inspect.signature(ref).parameters)
            assert list(inspect.signature(new).parameters)[:len(rp)] == rp, attr
        elif inspect.isclass(ref) and issubclass(ref, Exception):
            assert [c.__name__ for c in new.__mro__] == [c.__name__ for c in ref.__mro__], attr


def test_cp_init_hook_is_the_references(installed):
    import blockten.decomp as decomp

    saved = decomp._cp_init
    try:
        decomp._cp_init = lambda t, r: ("user hook", r)
        assert bt.decomp._cp_init(None, 3) == ("user hook", 3)
    finally:
        decomp._cp_init = saved


def test_uninstall_restores():
    import blockten.apps as apps
    import blockten.decomp as decomp

    before = (apps.hosvd, decomp.cp_als, blockten.errors.ShapeError, bt.decomp._cp_init)
    bt.install()
    bt.install()            # idempotent
    assert bt.installed() and apps.hosvd is bt.hosvd
    bt.uninstall()
    assert not bt.installed()
    assert (apps.hosvd, decomp.cp_als, blockten.errors.ShapeError, bt.decomp._cp_init) == before


def test_every_module_rebound_including_fileio(installed):
    """fileio raises ContainerFormatError / ShapeError that the CLI's
    except clauses (cli.py:385-392) must catch as bt200's classes."""
    import blockten.fileio as fileio

    assert "blockten.fileio" in installed
    assert fileio.ContainerFormatError is bt.ContainerFormatError
    assert fileio.ShapeError is bt.ShapeError


def test_cli_malformed_matrix_market_exit_code(installed, tmp_path, capsys):
    import blockten.cli as cli

    bad = tmp_path / "bad.mtx"
    bad.write_text("this is not a matrix market file\n1 2 3\n")
    code = cli.main(["analyze", str(bad), "--block-rows", "2", "--block-cols", "2"])
    assert code == 2, capsys.readouterr().err


def test_hook_set_before_install_is_honoured():
    import blockten.decomp as decomp

    saved = decomp._cp_init
    try:
        decomp._cp_init = lambda t, r: ("pre-install hook", r)
        bt.install()
        try:
            assert bt.decomp._cp_init(None, 5) == ("pre-install hook", 5)
            decomp._cp_init = saved          # the reference default -> bt200's HOSVD init
            assert bt.decomp._cp_init is not saved
        finally:
            bt.uninstall()
    finally:
        decomp._cp_init = saved
