import ctypes, sys, numpy as np, torch
sys.path.insert(0,'.')
from paper_2405_02520_b200 import _lib, make_plan
from paper_2405_02520_b200.abft import make_encoding
from paper_2405_02520_b200.fft_core import fit_group_size
from paper_2405_02520_b200.fft_core.plan import native_plan
lib=_lib.load()
for prec,logn,b in [("fp32",20,8),("fp32",17,16),("fp64",21,4),("fp32",14,64)]:
    n=1<<logn; td=torch.complex64 if prec=="fp32" else torch.complex128
    plan=fit_group_size(make_plan(n,prec,batch=b),b); h=native_plan(plan,0)
    row=make_encoding("wang",n).device_row(td,False)
    x=torch.randn((b,n),dtype=td,device="cuda"); y=torch.empty_like(x)
    rng=np.random.default_rng(5)
    for trial in range(6):
        f=_lib.Fault(); f.signal=int(rng.integers(b)); f.element=int(rng.integers(n)); f.component=int(rng.integers(2)); f.bit=30 if prec=="fp32" else 62; f.where=_lib.AT_OUTPUT
        rep=_lib.Report(); fl=(_lib.Flag*64)(); i64=ctypes.c_int64*64; cg,cs,ur=i64(),i64(),i64()
        rep.flagged,rep.flagged_cap=fl,64; rep.corrected_group,rep.corrected_signal,rep.corrected_cap=cg,cs,64; rep.unrecoverable,rep.unrecoverable_cap=ur,64
        _lib.check(lib.tfft_run_protected(h.handle,x.data_ptr(),y.data_ptr(),b,3,1e-4 if prec=="fp32" else 1e-9,0.0,row.data_ptr(),None,ctypes.byref(f),0,ctypes.byref(rep),torch.cuda.current_stream().cuda_stream),"run")
        torch.cuda.synchronize()
        # reference value of the faulted element
        yv=torch.fft.fft(x[f.signal].to(torch.complex128))[f.element]
        print(prec,logn,"sig",f.signal,"el",f.element,"comp",f.component,"fired",rep.fault_fired,"flagged",rep.n_flagged,"corr",rep.n_corrected,"y",complex(yv))
