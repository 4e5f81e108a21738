"""Run prrp_schur_update several times on fresh copies of one C and print a digest per run
(kernel-level determinism check; PRRP_SCHUR_WSC=0 selects the warp-specialised kernel that
reads C in its epilogue).  usage: schur_determinism.py M N K [reps]"""
import ctypes
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_1208_2451_b200 import _lib
    M, N, K = (int(v) for v in sys.argv[1:4])
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 6
    lib = _lib.device_lib()
    g = torch.Generator(device="cuda").manual_seed(1)
    C0 = torch.randn(M, N, dtype=torch.float64, device="cuda", generator=g)
    L = torch.randn(K, M, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(K, N, dtype=torch.float64, device="cuda", generator=g)
    ref = (C0 - L.t() @ B)
    for r in range(reps):
        C = C0.clone()
        mx, err = ctypes.c_double(0), _lib.PrrpErr()
        rc = lib.prrp_schur_update(ctypes.c_void_p(C.data_ptr()), N, ctypes.c_void_p(L.data_ptr()), M,
                                   ctypes.c_void_p(B.data_ptr()), N, M, N, K, ctypes.byref(mx), ctypes.byref(err),
                                   _lib.stream_handle())
        torch.cuda.synchronize()
        assert rc == 0
        d = (C - ref).abs().max().item()
        bad = int(((C - ref).abs() > 1e-9).sum().item())
        print(f"run {r}: digest {hashlib.sha1(C.cpu().numpy().tobytes()).hexdigest()[:12]} max|C - ref| {d:.3e} "
              f"elements off by > 1e-9: {bad}", flush=True)
        if bad:
            analyse(C, ref, C0, L, B, K)


def analyse(C, ref, C0, L, B, K):
    """Describe the wrong 8-row x 32-column strips of one run and look for the source of the operand
    they were computed with: err = (a_right - a_used)^T B_chunk, solved for a_used per k-chunk."""
    import torch
    M, N = C.shape
    bad = (C - ref).abs() > 1e-9
    strips = {}
    for r, c in bad.nonzero().tolist():
        strips.setdefault((r // 8, c // 32), 0)
        strips[(r // 8, c // 32)] += 1
    print(f"  {len(strips)} strips (8 rows x 32 columns): {sorted(strips.items())[:6]}")
    ntN = (N + 63) // 64
    for (rg, cg), cnt in sorted(strips.items())[:4]:
        R = slice(8 * rg, 8 * rg + 8)
        Cc = slice(32 * cg, 32 * cg + 32)
        err = (C - ref)[R, Cc]                                # 8 x 32
        tile = (8 * rg // 128) * ntN + (32 * cg) // 64
        print(f"  strip rows {8 * rg}..{8 * rg + 7} cols {32 * cg}..{32 * cg + 31}: tile {tile} (CTA {tile % 148}, its "
              f"tile #{tile // 148}), row group {(8 * rg % 128) // 8} of the tile; |err| {err.abs().max().item():.3e}")
        # C path: C_kernel = C_read - acc  =>  C_read = C_kernel + L^T B; where does C_read come from?
        c_read = C[R, Cc] + L[:, R].t() @ B[:, Cc]
        for name, src in (("the input C", C0), ("the updated C (ref)", ref)):
            dcol = (src[:, Cc] - c_read[:1, :]).abs().max(dim=1).values
            j = int(dcol.argmin().item())
            if dcol[j].item() < 1e-7:
                print(f"    C rows of this strip were READ from {name} rows {j}.. (same columns)")
        for q in range(K // 32):
            ks = slice(q * 32, (q + 1) * 32)
            Bq = B[ks, Cc]                                    # 32 x 32
            try:
                d = torch.linalg.solve(Bq.t(), err.t()).t()   # (a_right - a_used)^T, 8 x 32
            except Exception:
                continue
            a_used = L[ks, R] - d.t()                         # 32 x 8
            resid = (err - (L[ks, R] - a_used).t() @ Bq).abs().max().item()
            # where does a_used come from?
            if a_used.abs().max().item() < 1e-6:
                print(f"    k-chunk {q}: consistent with a ZERO operand (resid {resid:.1e})")
                continue
            diff = (L[ks, :] - a_used[:, :1]).abs().max(dim=0).values     # per row of L
            j = int(diff.argmin().item())
            if diff[j].item() < 1e-6:
                whole = (L[ks, j:j + 8] - a_used).abs().max().item() if j + 8 <= M else float("nan")
                tj = (j // 128)
                print(f"    k-chunk {q}: the operand used is L rows {j}..{j + 7} (tile row {tj}, row group {(j % 128) // 8}); "
                      f"all 8 rows match: {whole:.1e}")


if __name__ == "__main__":
    main()
