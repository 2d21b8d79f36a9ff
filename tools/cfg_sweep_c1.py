import os, subprocess, sys
for cfg in ["0", "2", "10", "11", "12"]:
    env = dict(os.environ, EB_CFG=cfg)
    r = subprocess.run([sys.executable, "-c", """
import ctypes, torch, sys
sys.path.insert(0, '/root/repo')
from paper_2206_08301_b200 import _capi as C
dev='cuda'
r=lambda *s: torch.rand(*s, dtype=torch.float64, device=dev)
X=r(512,512,512); B=r(512,24); Cm=r(512,24); out=torch.zeros(512,24,dtype=torch.float64,device=dev)
d=C.ContractDesc(); d.variant,d.mode,d.P,d.M,d.Q,d.L,d.R=C.EB_ROW,C.EB_REDUCE,1,512,512,512,24
d.X,d.U,d.ldu=X.data_ptr(),Cm.data_ptr(),24
d.n_pre=0; d.n_mid=1; d.mid[0]=C.Factor(B.data_ptr(),512,24)
d.out=out.data_ptr()
L=C.lib(); wb=L.eb_contract_workspace(ctypes.byref(d)); ws=torch.empty(wb,dtype=torch.uint8,device=dev)
st=ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3): C.check(L.eb_contract(ctypes.byref(d),ctypes.c_void_p(ws.data_ptr()),wb,st))
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(10): C.check(L.eb_contract(ctypes.byref(d),ctypes.c_void_p(ws.data_ptr()),wb,st))
e1.record(); torch.cuda.synchronize()
ms=e0.elapsed_time(e1)/10
want=torch.einsum('ijk,ja,ka->ia',X,B,Cm)
print(ms, 2*512**3*24/ms/1e9, ((out-want).norm()/want.norm()).item())
"""], env=env, capture_output=True, text=True)
    print(cfg, r.stdout.strip(), r.stderr.strip()[-300:])
