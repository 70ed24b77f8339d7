"""Timing of BASELINE configs 3, 4, 5 (single long series decompose, matvec and
Hankelization microbenchmarks) -- exploration script."""
import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_0911_4498_b200 as P, ssa_inputs
which = sys.argv[1:] or ["cfg4", "cfg5", "cfg3"]
ev = lambda: torch.cuda.Event(enable_timing=True)
if "cfg4" in which:
    N, L, B = 8192, 4096, 65536
    K = N - L + 1
    g = torch.Generator(device="cuda").manual_seed(4)
    F = torch.randn(B, N, dtype=torch.float64, device="cuda", generator=g)
    v = torch.randn(B, K, dtype=torch.float64, device="cuda", generator=g)
    u = torch.randn(B, L, dtype=torch.float64, device="cuda", generator=g)
    plan = P.Plan(N, L, 0, B)
    spec = plan.spectrum(F); y = torch.empty(B, L, dtype=torch.float64, device="cuda"); z = torch.empty(B, K, dtype=torch.float64, device="cuda")
    for _ in range(2):
        plan.matvec(spec, v, out=y); plan.matvec(spec, u, transpose=True, out=z)
    torch.cuda.synchronize()
    a, b = ev(), ev(); a.record()
    for t in range(64):
        if t % 2 == 0: plan.matvec(spec, v, out=y)
        else: plan.matvec(spec, u, transpose=True, out=z)
    b.record(); torch.cuda.synchronize(); ms = a.elapsed_time(b)
    nprod = 64 * B
    byt = nprod * (8 * (K + L) + 16 * (N // 2 + 1))
    print(f"cfg4: {ms:.1f} ms for {nprod} products -> {nprod/ms/1e3:.2f} M products/s, {byt/ms/1e6:.0f} GB/s algorithmic")
    del F, v, u, spec, y, z, plan
if "cfg5" in which:
    N, L, B, T = 262144, 131072, 256, 50
    K = N - L + 1
    g = torch.Generator(device="cuda").manual_seed(5)
    Bc = 32
    U = torch.randn(Bc, T, L, dtype=torch.float64, device="cuda", generator=g); U /= U.norm(dim=2, keepdim=True)
    V = torch.randn(Bc, T, K, dtype=torch.float64, device="cuda", generator=g); V /= V.norm(dim=2, keepdim=True)
    sig = (1.0 / torch.arange(1, T + 1, dtype=torch.float64, device="cuda")).repeat(Bc, 1).contiguous()
    plan = P.Plan(N, L, 0, Bc)
    out = torch.empty(Bc, T, N, dtype=torch.float64, device="cuda")
    plan.hankelize(sig, U, V, out=out); torch.cuda.synchronize()
    a, b = ev(), ev(); a.record()
    plan.hankelize(sig, U, V, out=out)
    b.record(); torch.cuda.synchronize(); ms = a.elapsed_time(b)
    nt = Bc * T
    print(f"cfg5: {ms:.1f} ms for {nt} terms -> {nt/ms*1e3:.0f} terms/s ({ms/nt*1e3:.1f} us/term)")
    del U, V, out, plan
if "cfg3" in which:
    f = ssa_inputs.cfg3_series()
    N, L, k = 1 << 20, 1 << 19, 32
    plan = P.Plan(N, L, k, 1, profile=False)
    x = torch.from_numpy(f[None].copy()).cuda()
    s, U, V, info = plan.decompose(x); torch.cuda.synchronize()
    t0 = time.time()
    a, b = ev(), ev(); a.record()
    s, U, V, info = plan.decompose(x, s, U, V, info)
    b.record(); torch.cuda.synchronize(); ms = a.elapsed_time(b)
    inf = P.info_to_numpy(info)[0]
    print(f"cfg3: {ms:.1f} ms (wall {1e3*(time.time()-t0):.1f}) steps {inf['steps']} status {inf['status']} res {inf['max_residual']:.2e} -> {k/ms*1e3:.0f} triples/s")
    print("sigma", s.cpu().numpy()[0][:6])
