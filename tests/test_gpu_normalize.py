"""The normalisation prepass on the device (htr_normalize / htr_denormalize,
metrics.hpp:93-197) against a restatement of the reference's host
algorithm: per-field parameters (maxima exact; sums to 1e-15 relative, the
reference sums sequentially), scaled tensors, floored constant fields, the
inverse, and every field layout (no axis, first / middle / last mode, more
fields than one accumulation pass holds)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ht():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2412_16544_b200 import htrise

    htrise.set_default_context(htrise.Context(0))
    return htrise


def reference_normalize(y, method, axis):
    """metrics.hpp:93-171 restated (numpy, per field)."""
    fields = 1 if axis is None else y.shape[axis]
    sl = (lambda f: y) if axis is None else (lambda f: np.take(y, f, axis=axis))
    scale, offset, floored = np.zeros(fields), np.zeros(fields), [False] * fields
    for f in range(fields):
        v = sl(f).ravel()
        if method == "maxabs":
            scale[f] = np.max(np.abs(v))
        elif method == "unitvec":
            scale[f] = np.sqrt(np.sum(v * v))
        elif method == "zscore":
            offset[f] = np.sum(v) / v.size
            scale[f] = np.sqrt(np.sum((v - offset[f]) ** 2) / v.size)
        else:
            scale[f] = 1.0
        if scale[f] == 0.0:
            scale[f], floored[f] = 1.0, True
    shape = [1] * y.ndim
    if axis is not None:
        shape[axis] = fields
    out = (y - (offset.reshape(shape) if method == "zscore" else 0.0)) / scale.reshape(shape)
    return out, scale, offset, floored


@pytest.mark.parametrize("method", ["maxabs", "unitvec", "zscore", "none"])
@pytest.mark.parametrize("shape,axis", [((6, 7, 5, 3), None), ((6, 7, 5, 3), 0), ((6, 7, 5, 3), 2),
                                        ((5, 4, 40, 3), 2), ((9, 8, 2), 1)])
def test_normalize_matches_reference(ht, method, shape, axis):
    rng = np.random.default_rng(abs(hash((method, shape, axis))) % 2**32)
    y = np.asfortranarray(3.0 + rng.standard_normal(shape) * rng.uniform(0.5, 5.0, size=shape[-1]))
    if axis is not None:  # one constant field (floored scale for zscore)
        idx = [slice(None)] * len(shape)
        idx[axis] = 1
        y[tuple(idx)] = 2.5
    got, p = ht.normalize(y, method, axis)
    want, sc, off, fl = reference_normalize(y, method, axis)
    if method == "maxabs":
        assert p.scale == list(sc)
    else:
        assert np.allclose(p.scale, sc, rtol=1e-14, atol=0)
        assert np.allclose(p.offset, off, rtol=1e-14, atol=1e-15)
    assert p.floored == fl
    assert np.allclose(got, want, rtol=1e-13, atol=1e-13)
    back = ht.denormalize(got, p)
    assert np.allclose(back, y, rtol=1e-13, atol=1e-12)


def test_normalize_device_batch_in_place(ht):
    import torch

    rng = np.random.default_rng(3)
    y = np.asfortranarray(rng.standard_normal((16, 16, 8, 4)))
    t = torch.from_numpy(np.ascontiguousarray(y.transpose())).cuda().reshape(-1)
    d = ht.DeviceTensor(t, y.shape)
    _, p = ht.normalize(d, "unitvec", 2)
    want, sc, _, _ = reference_normalize(y, "unitvec", 2)
    back = t.cpu().numpy().reshape(tuple(reversed(y.shape))).transpose()
    assert np.allclose(back, want, rtol=1e-13, atol=1e-13)
    assert np.allclose(p.scale, sc, rtol=1e-14)
