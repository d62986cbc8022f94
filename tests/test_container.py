"""The container format (container.py:1-346, blockten-container/1) against
files written by the unmodified reference (tests/golden/containers/*.btc,
make_golden.py:container_cases).  CPU: header/payload validation and error
semantics (they fire before any device work).  GPU: read -> write reproduces
the reference's bytes for every representation kind; arrays decode exactly."""

import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN

CDIR = os.path.join(GOLDEN, "containers")
KINDS = ("kron_sum", "blr", "tucker_raw", "spsd", "spd", "multilevel")


def _decode(blob):
    """Test-side numpy decode of the payload (first-index-fastest float64)."""
    head, payload = blob.split(b"\n---\n", 1)
    kv = dict(l.split(": ", 1) for l in head.decode().split("\n")[1:] if l)
    out, pos = {}, 0
    for name in kv["arrays"].split():
        nd = int(np.frombuffer(payload, "<i8", 1, pos)[0])
        ext = tuple(int(e) for e in np.frombuffer(payload, "<i8", nd, pos + 8))
        pos += 8 * (1 + nd)
        cnt = int(np.prod(ext))
        out[name] = np.frombuffer(payload, "<f8", cnt, pos).reshape(ext, order="F")
        pos += 8 * cnt
    return kv, out


def test_container_kind_and_errors_cpu(tmp_path):
    from paper_2105_01170_b200 import container
    from paper_2105_01170_b200.errors import ContainerExtentError, ContainerFormatError

    for kind in KINDS:
        assert container.container_kind(os.path.join(CDIR, f"{kind}.btc")) == kind
    blob = open(os.path.join(CDIR, "kron_sum.btc"), "rb").read()

    def write(name, data):
        p = tmp_path / name
        p.write_bytes(data)
        return p

    with pytest.raises(ContainerFormatError):
        container.container_read(write("v2.btc", blob.replace(b"container/1", b"container/2", 1)))
    with pytest.raises(ContainerFormatError):
        container.container_read(write("nosep.btc", blob.replace(b"\n---\n", b"\n--\n", 1)))
    with pytest.raises(ContainerFormatError):
        container.container_read(write("trunc.btc", blob[:-9]))
    with pytest.raises(ContainerFormatError):
        container.container_read(write("trail.btc", blob + b"\0" * 8))
    head, payload = blob.split(b"\n---\n", 1)
    # corrupt the first array's rank prefix -> extent error
    bad = head + b"\n---\n" + np.array([9], "<i8").tobytes() + payload[8:]
    with pytest.raises(ContainerExtentError):
        container.container_read(write("rank.btc", bad))
    # header extents disagreeing with the payload prefix
    kv, _ = _decode(blob)
    first = kv["arrays"].split()[0]
    spec = kv[f"array.{first}"]
    bad = blob.replace(f"array.{first}: {spec}".encode(),
                       f"array.{first}: {spec} 1".encode(), 1)
    with pytest.raises(ContainerExtentError):
        container.container_read(write("ext.btc", bad))
    dup = blob.replace(b"kind: kron_sum", b"kind: kron_sum\nkind: kron_sum", 1)
    with pytest.raises(ContainerFormatError):
        container.container_read(write("dup.btc", dup))


@pytest.mark.gpu
@pytest.mark.parametrize("kind", KINDS)
def test_container_read_write_bit_identical(kind, tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("needs a CUDA device")
    import paper_2105_01170_b200 as bt

    src = os.path.join(CDIR, f"{kind}.btc")
    ref = open(src, "rb").read()
    rep = bt.container_read(src)
    out = tmp_path / "again.btc"
    kv, arrays = _decode(ref)
    seed = int(kv["seed"]) if "seed" in kv else None
    ranks = tuple(int(r) for r in kv["ranks"].split()) if "ranks" in kv else None
    bt.container_write(out, rep, seed=seed, ranks=ranks)
    assert out.read_bytes() == ref
    # device arrays round-trip too (one H2D per array, layout flip on the GPU)
    rep_d = bt.container_read(src, device=True)
    bt.container_write(tmp_path / "dev.btc", rep_d, seed=seed, ranks=ranks)
    assert (tmp_path / "dev.btc").read_bytes() == ref
    if kind == "kron_sum":
        assert np.array_equal(rep.coeffs, arrays["coeffs"])
        assert np.array_equal(rep.terms, arrays["terms"])
        x = np.random.default_rng(1).standard_normal(rep.pattern.shape[1])
        assert np.allclose(bt.matvec(rep, x), bt.densify(rep) @ x, rtol=1e-12, atol=1e-12)
    if kind == "spd":
        assert np.array_equal(rep.chol, arrays["chol"])
        d = rep.densify()
        assert np.allclose(d, d.T, atol=1e-12)
    if kind == "multilevel":
        assert rep.pattern.depth == 2
        # densify == ml_tensor_to_mat of the reconstruction (restated here in numpy)
        from oracle import port

        core = arrays["core"]
        recon = core
        for k in range(core.ndim):
            recon = port.mode_multiply(recon, k + 1, arrays[f"factor{k + 1}"])
        outer, inner = rep.pattern.levels

        def assemble(pat, items):           # items[k]: class k's block
            out = np.zeros(pat.shape)
            for k, cells in enumerate(pat.placements):
                for i, j in cells:
                    out[i * pat.m:(i + 1) * pat.m, j * pat.n:(j + 1) * pat.n] = (
                        items[k] / np.sqrt(len(cells)))
            return out

        inner_mats = [assemble(inner, [recon[:, k1, k2, :] for k2 in range(inner.p)])
                      for k1 in range(outer.p)]
        want = assemble(outer, inner_mats)
        assert np.allclose(rep.densify(), want, rtol=0, atol=1e-12 * np.abs(want).max())
