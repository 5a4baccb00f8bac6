"""The `b200` operator table against the reference's own operator I/O
(golden vectors from the NumPy backend), at bf16 tolerance."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


def test_table_surface(cuda):
    from paper_2512_23379_b200 import ftlk_backend as B
    for name in ("dense_forward", "dense_backward", "gelu_forward", "gelu_backward", "layernorm_forward",
                 "layernorm_backward", "mha_forward", "mha_backward"):
        assert callable(getattr(B, name))
    assert B.NAME == "b200"
    with pytest.raises(NotImplementedError):
        B.dense_backward(None, None, None)


def test_dense_gelu_layernorm(golden, cuda):
    from paper_2512_23379_b200 import ftlk_backend as B
    g = golden
    assert rel(B.dense_forward(g["k_dense_x"], g["k_dense_w"], g["k_dense_b"]), g["k_dense_y"]) < 1e-2
    assert rel(B.gelu_forward(g["k_gelu_x"]), g["k_gelu_y"]) < 1e-2
    y, mu, rs = B.layernorm_forward(g["k_ln_x"], g["k_ln_g"], g["k_ln_b"])
    assert rel(y, g["k_ln_y"]) < 1e-2
    assert rel(mu, g["k_ln_mean"]) < 1e-6 and rel(rs, g["k_ln_rstd"]) < 1e-6


@pytest.mark.parametrize("heads", [1, 2, 4])
@pytest.mark.parametrize("cross", [0, 1])
def test_mha(golden, cuda, heads, cross):
    from paper_2512_23379_b200 import ftlk_backend as B
    k = "k_mha_h%d_c%d_" % (heads, cross)
    y, cache = B.mha_forward(golden[k + "xq"], golden[k + "xkv"], golden[k + "wq"], golden[k + "wk"],
                             golden[k + "wv"], golden[k + "wo"], heads)
    assert rel(y, golden[k + "y"]) < 2e-2
    assert cache[0].shape == (heads, 5, 8 // heads)
