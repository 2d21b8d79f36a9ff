import ctypes, json, os, subprocess, sys
sys.path.insert(0, "/root/repo")
for cfg in ["0", "2", "10", "11", "12", "13"]:
    env = dict(os.environ, EB_CFG=cfg)
    r = subprocess.run([sys.executable, "-c", """
import ctypes, torch, sys
sys.path.insert(0, '/root/repo')
from paper_2206_08301_b200 import _capi as C
dev='cuda'
r=lambda *s: torch.rand(*s, dtype=torch.float64, device=dev)
X=r(64,64,64,64,64); F=[r(64,24) for _ in range(4)]; out=torch.zeros(64,24,dtype=torch.float64,device=dev)
d=C.ContractDesc(); d.variant,d.mode,d.P,d.M,d.Q,d.L,d.R=C.EB_ROW,C.EB_REDUCE,1,64,64**3,64,24
d.X,d.U,d.ldu=X.data_ptr(),F[3].data_ptr(),24
d.n_pre=0; d.n_mid=3
for i in range(3): d.mid[i]=C.Factor(F[i].data_ptr(),64,24)
d.out=out.data_ptr()
L=C.lib(); wb=L.eb_contract_workspace(ctypes.byref(d)); ws=torch.empty(wb,dtype=torch.uint8,device=dev)
st=ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3): C.check(L.eb_contract(ctypes.byref(d),ctypes.c_void_p(ws.data_ptr()),wb,st))
ref=out.clone()
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(5): C.check(L.eb_contract(ctypes.byref(d),ctypes.c_void_p(ws.data_ptr()),wb,st))
e1.record(); torch.cuda.synchronize()
ms=e0.elapsed_time(e1)/5
# correctness vs torch einsum
want=torch.einsum('ijklm,ja,ka,la,ma->ia',X,F[0],F[1],F[2],F[3])
err=((out-want).norm()/want.norm()).item()
print(ms, 2*64**5*24/ms/1e9, err)
"""], env=env, capture_output=True, text=True)
    print(cfg, r.stdout.strip(), r.stderr.strip()[-300:])
