"""Print bf16/fp32 parity errors per case (development diagnostic)."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import test_gpu_parity as T

for case in T.FB_CASES + T.TINY_CASES:
    for prec in ["bf16"]:
        res = T._run_single(case, prec)
        for (L, Lr, gx, gxr, dW, dWr, Wn, Wnr, Vn, Vnr) in res:
            print(case, prec, f"L={Lr:.4g} relL={abs(L-Lr)/abs(Lr):.2e} gx={T.maxrel(gx,gxr):.2e} dW={T.maxrel(dW,dWr):.2e} V={T.maxrel(Vn,Vnr):.2e}", flush=True)
