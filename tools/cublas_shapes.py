import torch, time
torch.backends.cuda.matmul.allow_tf32=False
def t(M,N,K,ta=False,reps=10):
    A = torch.randn(K,M,dtype=torch.float64,device='cuda').T if not ta else torch.randn(M,K,dtype=torch.float64,device='cuda')
    # column-major A (M x K): stored as K x M row-major -> .T
    B = torch.randn(N,K,dtype=torch.float64,device='cuda').T
    for _ in range(3): C = A @ B
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): C = A @ B
    e1.record(); torch.cuda.synchronize()
    ms=e0.elapsed_time(e1)/reps
    print(f"cublas {M}x{N}x{K} ta={ta}: {ms:.3f} ms {2*M*N*K/ms/1e9:.2f} TF/s",flush=True)
t(40960,320,1000); t(320,1000,40960,True); t(320,128000,1000); t(1000,320,128000); t(8192,8192,8192,reps=3)
t(40960,288,32); t(32,288,40960,True)
