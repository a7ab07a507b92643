"""Fixed cost of one BLOCK solve (trace build: python tools/build_variant.py trace -DSPTRSV_BLOCK_TRACE=1,
SPTRSV_DEV_LIB=paper_1710_04985_b200/lib/var_trace.so): CUDA-event time of the solve vs kernel
entry -> first step -> last step -> loop exit (%globaltimer, per warp).
usage: python tools/overhead.py DIMS [DIMS ...]   e.g. 8x4x128 128x128x128"""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
from paper_1710_04985_b200 import sptrsv as S

lib = ctypes.CDLL(S.LIB_PATH)
lib.sptrsv_dbg_block_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
lib.sptrsv_dbg_block_plan.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
for spec in sys.argv[1:]:
    dims = tuple(int(v) for v in spec.split("x"))
    m = workloads.stencil(dims, 7, "lower")
    sv = S.from_csr(m, algo="block")
    out = (ctypes.c_longlong * 13)()
    lib.sptrsv_dbg_block_plan(ctypes.c_void_p(sv.handle), out)
    U = out[0] * out[1]
    cap = 4096
    b = torch.from_numpy(workloads.rhs(m.n, 1, seed=2)[:, 0]).cuda()
    x = torch.empty_like(b)
    buf = torch.zeros(U * cap, dtype=torch.int64, device="cuda")
    lib.sptrsv_dbg_block_trace(ctypes.c_void_p(sv.handle), ctypes.c_void_p(buf.data_ptr()), cap)
    for _ in range(3):
        sv.solve(b, x)
    torch.cuda.synchronize()
    ev = []
    rows = []
    for _ in range(5):
        buf.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); sv.solve(b, x); e1.record(); e1.synchronize()
        ev.append(e0.elapsed_time(e1) * 1e3)
        tr = buf.view(U, cap).cpu().numpy().astype(np.int64)
        live = tr[:, cap - 1] > 0
        tr = tr[live]
        entry, exit_ = tr[:, cap - 2], tr[:, cap - 1]
        first = tr[:, 0]
        nst = (tr[:, :cap - 8] > 0).sum(1)
        nc, nf, npend = tr[:, cap - 3], tr[:, cap - 4], tr[:, cap - 5]
        last = tr[np.arange(len(tr)), np.maximum(nst - 1, 0)]
        t0 = entry.min()
        late = (nc.sum() / nst.sum(), nf.sum() / nst.sum(), npend.sum() / nst.sum(), nc[0], nf[0], npend[0], nst[0])
        rows.append(((entry - t0).max() / 1e3, (first - entry).mean() / 1e3, (first - t0).min() / 1e3,
                     (last - t0).max() / 1e3, (exit_ - t0).max() / 1e3, np.median((last - first) / np.maximum(nst - 1, 1))))
    r = np.median(np.array(rows), axis=0)
    os.makedirs("gpurun_out", exist_ok=True)
    np.savez_compressed(f"gpurun_out/oh_{spec}.npz", tr=buf.view(U, cap).cpu().numpy(), plan=np.array(list(out)),
                        nlev=sv.info()["nlev"], dims=np.array(dims))
    print(f"{spec}: nlev {sv.info()['nlev']} warps {U}: event {np.median(ev):.1f} us | entry spread {r[0]:.2f} us, "
          f"entry->first step {r[1]:.2f} us (min from first entry {r[2]:.2f}), last step {r[3]:.1f} us, "
          f"last loop exit {r[4]:.1f} us after first entry; median ns/step per warp {r[5]:.0f}")
    print(f"   steps with ctl ring late {late[0]:.3f}, coef ring late {late[1]:.3f}, EXT pending {late[2]:.3f} "
          f"(warp 0: {late[3]}/{late[4]}/{late[5]} of {late[6]} steps)")
    cb, csl, ctot = tr[:, cap - 6].astype(float), tr[:, cap - 7].astype(float), tr[:, cap - 8].astype(float)
    print(f"   loop cycles: b wait {cb.sum() / ctot.sum():.3f}, slow path {csl.sum() / ctot.sum():.3f} of the total; "
          f"per step: total {ctot.sum() / nst.sum():.0f}, b wait {cb.sum() / nst.sum():.0f}, slow {csl.sum() / nst.sum():.0f} cycles")
    sv.close()
