"""Stream re-entrancy of the C ABI (SURVEY §8(b) "apply/spmv are re-entrant
across streams with distinct outputs"): work issued concurrently on two
CUDA streams gives results bit-identical to the same work run serially.

* two MG-FGMRES solves (two hierarchies, each with its own Krylov workspace
  and reduction scratch) driven from two host threads, one stream each;
* two sweeps of ONE patch set on two streams, each with its own correction
  buffer (``zbuf``), interleaved launch by launch.
"""

import threading

import numpy as np
import pytest

from conftest import load_case

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.mark.parametrize("name", ["s_thtri2", "s_bdm3"])
def test_two_fgmres_solves_on_two_streams(name):
    import torch
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200.solver import FgmresSolver, mg_rhs
    pack, _ = load_case(name)
    b1 = mg_rhs(pack)
    b2 = np.random.default_rng(7).uniform(-1.0, 1.0, b1.size)
    b2[np.asarray(pack.fine.system.bc.indices)] = 0.0
    solvers = [FgmresSolver(V.hierarchy_from_pack(pack)) for _ in range(2)]
    rhs = [b1, b2]
    # serial reference (also captures every step graph of both solvers)
    serial = [solvers[k].solve(rhs[k]) for k in range(2)]
    out = [None, None]
    err = []
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    go = threading.Barrier(2)

    def work(k):
        try:
            with torch.cuda.stream(streams[k]):
                go.wait()
                for _ in range(3):
                    out[k] = solvers[k].solve(rhs[k])
                streams[k].synchronize()
        except Exception as e:  # pragma: no cover - surfaced below
            err.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not err, err
    for k in range(2):
        x_s, its_s, conv_s, hist_s = serial[k]
        x_c, its_c, conv_c, hist_c = out[k]
        assert its_c == its_s and conv_c == conv_s
        assert np.array_equal(_bits(hist_c), _bits(hist_s))
        assert np.array_equal(_bits(x_c), _bits(x_s))


@pytest.mark.parametrize("name", ["cfg1", "s_thtri4"])
def test_two_sweeps_of_one_patch_set_on_two_streams(name):
    import torch
    import paper_2409_14222_b200 as V
    from paper_2409_14222_b200 import _lib as L
    pack, _ = load_case(name)
    lv = pack.fine
    ps = V.factor_patches(V.build_patches(lv.mixed, lv.system.bc), lv.system)
    n = lv.system.matrix.shape[0]
    rng = np.random.default_rng(11)
    rs = [torch.from_numpy(rng.uniform(-1, 1, n)).cuda() for _ in range(2)]
    serial = [V.apply_additive(ps, r).clone() for r in rs]
    torch.cuda.synchronize()
    zb = [ps.new_zbuf() for _ in range(2)]
    outs = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in range(2)]
    s = [torch.cuda.Stream(), torch.cuda.Stream()]
    for _ in range(20):
        for k in range(2):            # interleaved: both streams in flight
            L.call("vk_patches_apply", ps.handle, L.ptr(rs[k]), L.ptr(outs[k]), 1.0,
                   L.VK_APPLY_OUT, L.ptr(zb[k]), s[k].cuda_stream)
    torch.cuda.synchronize()
    for k in range(2):
        assert torch.equal(outs[k], serial[k])


def test_zbuf_size_is_checked():
    import torch
    import paper_2409_14222_b200 as V
    pack, _ = load_case("cfg1")
    lv = pack.fine
    ps = V.factor_patches(V.build_patches(lv.mixed, lv.system.bc), lv.system)
    r = torch.zeros(lv.system.matrix.shape[0], dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        V.apply_additive(ps, r, zbuf=torch.empty(3, dtype=torch.float64, device="cuda"))
