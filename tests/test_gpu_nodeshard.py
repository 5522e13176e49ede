"""One GEP split by quadrature node over two ranks (dist.solve_multi_node_sharded), the ranks being two
host threads with their own streams on the one GPU a test box has; the all-reduce is done on the host
side of the test (no kernel of one rank waits for the other: each rank synchronises its stream first).
Both ranks must return the eigenpairs of the unsharded solve."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


class HostAllReduce:
    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world
        self.result = None

    def rank_fn(self, rank):
        def run(t, op):
            torch.cuda.current_stream().synchronize()
            self.slots[rank] = t
            self.barrier.wait(timeout=300)
            if rank == 0:
                acc = self.slots[0].clone()
                for r in range(1, self.world):
                    acc = acc + self.slots[r] if op == "sum" else torch.minimum(acc, self.slots[r])
                torch.cuda.current_stream().synchronize()
                self.result = acc
            self.barrier.wait(timeout=300)
            t.copy_(self.result)
            torch.cuda.current_stream().synchronize()
            self.barrier.wait(timeout=300)
        return run


def _run_sharded(pencil, contours, cfg, world=2, solver="cirr"):
    from paper_2511_01927_b200 import solvers as S
    from paper_2511_01927_b200.dist import solve_multi_node_sharded

    ar = HostAllReduce(world)
    out, errs = [None] * world, [None] * world

    def worker(rank):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                out[rank] = solve_multi_node_sharded(pencil, contours, cfg, solver, 0,
                                                     shard_ctx=S.NodeShard(rank, world, ar.rank_fn(rank)))
                torch.cuda.current_stream().synchronize()
        except BaseException as exc:  # noqa: BLE001 -- reported by the main thread
            errs[rank] = exc
            ar.barrier.abort()

    ths = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=600)
    for e in errs:
        if e is not None:
            raise e
    return out


@pytest.mark.parametrize("n,count", [(256, 8), (2048, 60)])   # 2048: int8 updates, factor slices per rank
def test_node_split_matches_unsharded(n, count):
    if not torch.cuda.is_available():
        pytest.fail("gpu test without CUDA")
    from paper_2511_01927_b200 import Contour, SolverConfig, solve_multi
    from paper_2511_01927_b200 import workloads as W

    a, b = W.config4_matrices(seed=3 if n == 256 else 0, n=n)

    class P:
        pass

    p = P()
    p.a, p.b, p.hermitian = a, b, False
    cs = [Contour(shape="ellipse", center=0.5 + 0j, semi_re=0.3, semi_im=0.15, expected_count=count),
          Contour(shape="ellipse", center=-0.5 + 0j, semi_re=0.3, semi_im=0.15, expected_count=count)]
    cfg = SolverConfig(n_q=32, source_cols=16, n_moments=4) if n == 256 else \
        SolverConfig(n_q=64, source_cols=32, n_moments=8)
    ref = solve_multi(p, cs, cfg, seed=0)
    got = _run_sharded(p, cs, cfg)
    assert len(ref.eigenvalues) > 0
    for m in got:
        assert [type(e) for e in m.errors] == [type(e) for e in ref.errors]
        assert len(m.eigenvalues) == len(ref.eigenvalues)
        for lam in ref.eigenvalues:
            assert np.min(np.abs(m.eigenvalues - lam)) <= 1e-9 * max(1.0, abs(lam))
        for r in m.results:
            if r is not None:
                assert r.residuals.max() <= 1e-10
                assert r.stats.n_factorizations == cfg.n_q // 2      # half of the nodes on each rank
    # the ranks ran the same Rayleigh-Ritz on the same sums: identical results
    assert np.array_equal(got[0].eigenvalues, got[1].eigenvalues)


def test_node_split_singular_shift_agreed():
    """A singular shift seen by one rank drops the contour on both (min-reduction after the factorisation)."""
    if not torch.cuda.is_available():
        pytest.fail("gpu test without CUDA")
    from paper_2511_01927_b200 import Contour, SolverConfig
    from paper_2511_01927_b200.errors import SingularShiftError

    class P:
        pass

    p = P()
    p.a, p.b, p.hermitian = np.diag([1.0, 2.0, 3.0, 10.0]), np.eye(4), True
    # node 0 of the midpoint rule on this circle is not an eigenvalue; put an eigenvalue exactly on node 1's z:
    c = Contour(shape="circle", center=2.0 + 0j, radius=1.5, expected_count=3)
    from paper_2511_01927_b200.contours import quadrature_for
    z1 = complex(quadrature_for(c, 8).nodes[1])
    p.a = np.diag([z1.real, 2.0, 3.0, 10.0]).astype(np.complex128)
    p.a[0, 0] = z1
    p.hermitian = False
    got = _run_sharded(p, [c], SolverConfig(n_q=8, source_cols=4, n_moments=2))
    for m in got:
        assert isinstance(m.errors[0], SingularShiftError) and m.errors[0].node_index == 1
