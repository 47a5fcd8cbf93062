import ctypes, numpy as np, sys, time
sys.path.insert(0,'/root/repo')
from oracle import oracle as orc
L=ctypes.CDLL('/tmp/chain_sim.so')
f64p=ctypes.POINTER(ctypes.c_double); i64p=ctypes.POINTER(ctypes.c_int64); u32p=ctypes.POINTER(ctypes.c_uint32)
L.sim_predict.restype=ctypes.c_int64
L.sim_predict.argtypes=[f64p,ctypes.c_int64,ctypes.c_double,ctypes.c_int64,ctypes.c_int,ctypes.c_int,i64p,i64p]
L.sim_codes.restype=ctypes.c_int64
L.sim_codes.argtypes=[f64p,ctypes.c_int64,ctypes.c_double,ctypes.c_int64,u32p,f64p]
def pred(x, eb, L_=32, mode=0, nbh=32768):
    x=np.ascontiguousarray(x,dtype=np.float64); fb=ctypes.c_int64(); ne=ctypes.c_int64()
    bad=L.sim_predict(x.ctypes.data_as(f64p), x.size, eb, nbh, L_, mode, ctypes.byref(fb), ctypes.byref(ne))
    return bad, fb.value, ne.value, (x.size-1+L_-1)//L_
def sine(n, seed=0):
    r=np.random.default_rng(seed); f=r.uniform(1,64,8); a=r.uniform(0,1,8); p=r.uniform(0,2*np.pi,8)
    t=np.arange(n)/n
    out=np.zeros(n)
    for k in range(8): out+=a[k]*np.sin(2*np.pi*f[k]*t+p[k])
    return out + r.normal(0,1e-3,n)
z=np.load('/root/repo/tests/golden/golden.npz')
# lc_step parity with oracle on a few golden vectors
for name in ['sine_r6','jac190_r6','edge_1','crit6_3']:
    x=z[str(z[name+'/x'])]; cfg=z[name+'/cfg']
    vr=x.max()-x.min(); eb=cfg[1] if cfg[0]==0 else cfg[1]*vr
    c=np.empty(x.size-1,np.uint32); rc=np.empty(x.size)
    L.sim_codes(x.ctypes.data_as(f64p), x.size, eb, int(cfg[2]), c.ctypes.data_as(u32p), rc.ctypes.data_as(f64p))
    oc,orec,_,_,_=orc.compress_kernel(x,eb,int(cfg[2]))
    print(name, 'codes eq', np.array_equal(c.astype(np.int64),oc), 'recon eq', np.array_equal(rc.view(np.int64),orec.view(np.int64)))
n=1<<int(sys.argv[1]) if len(sys.argv)>1 else 1<<20
x=sine(n)
vr=x.max()-x.min()
for ebr in (1e-3,1e-4,1e-6):
    for mode in (0,1):
        t=time.time(); r=pred(x, ebr*vr, 32, mode); print('sine n=%d eb=%g mode=%d bad=%d first=%d events=%d chunks=%d  %.1fs'%(n,ebr,mode,*r,time.time()-t))
for name in ['jac190_r4','jac190_r6','sine_r6','edge_0','ident_25_r6','crit6_2']:
    x=z[str(z[name+'/x'])]; cfg=z[name+'/cfg']
    vr=x.max()-x.min(); eb=cfg[1] if cfg[0]==0 else cfg[1]*vr
    print(name, pred(x, eb, 32, 0, int(cfg[2])), pred(x,eb,32,1,int(cfg[2]))[:2])
