"""Quick timing probe on one GPU: setup + solve at a few sizes (development aid)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2303_02352_b200 as pb  # noqa: E402


def run(stencil, nd, reps=2):
    n = nd ** 3
    rt = pb.Runtime(0, 0, 1)
    t0 = time.time()
    nnz = pb.lib().pairamg_poisson_nnz(stencil, nd, nd, nd, 0, n)
    rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    ci = torch.empty(nnz, dtype=torch.int64, device="cuda")
    va = torch.empty(nnz, dtype=torch.float64, device="cuda")
    pb._check(pb.lib().pairamg_poisson_device(rt.h, stencil, nd, nd, nd, 0, n, pb._ptr(rp), pb._ptr(ci), pb._ptr(va)))
    torch.cuda.synchronize()
    tg = time.time() - t0
    s = pb.Solver(rt)
    for _ in range(reps):
        t0 = time.time()
        s.setup(n, [0, n], rp, ci, va, cfg=pb.SetupConfig(3, 40 * nd, 40))
        ts = time.time() - t0
    st_ = s.setup_stats()
    b = torch.ones(n, dtype=torch.float64, device="cuda")
    for _ in range(reps):
        u = torch.zeros(n, dtype=torch.float64, device="cuda")
        st = s.solve(b, u)
    s.set_kernel_timing(True)
    u = torch.zeros(n, dtype=torch.float64, device="cuda")
    st2 = s.solve(b, u)
    kt = [s.kernel_timing(k) for k in range(4)]
    print(f"{stencil}pt {nd}^3 gen={tg:.3f}s setup={ts:.3f}s ({ {k: round(v, 4) if isinstance(v, float) else v for k, v in st_.items()} }) "
          f"levels={s.level_sizes()} iters={st.iterations} relres={st.final_relres:.3e} solve={st.t_solve_s*1e3:.2f}ms "
          f"ms/iter={st.t_solve_s*1e3/st.iterations:.3f} launches={s.launch_count()}")
    for k, name in enumerate(["L0 sweep", "L0 resid", "L0 spmv+dots", "update", "L0 zero-sweep fused", "L0 prolong-sweep fused"]):
        t = kt[k]
        if t["launches"]:
            avg = t["ms"] / t["launches"]
            print(f"   {name}: {t['launches']} launches avg {avg*1e3:.1f}us  {t['bytes_per_launch']/avg/1e6:.0f} GB/s")
    print(f"   timed-solve ms/iter={st2.t_solve_s*1e3/st2.iterations:.3f}")
    s.close()
    rt.close()


if __name__ == "__main__":
    for arg in sys.argv[1:] or ["7:64", "7:128", "7:256", "27:192"]:
        st, nd = arg.split(":")
        run(int(st), int(nd))
