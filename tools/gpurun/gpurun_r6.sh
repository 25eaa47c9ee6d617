cd $GRAFT_REPO_ROOT
python tools/gemm_bench.py > gpurun_out/r6_gemm.log 2>&1
python -c "
import torch,time
a=torch.randn(8192,8192,dtype=torch.float64,device='cuda');b=torch.randn(8192,8192,dtype=torch.float64,device='cuda')
for i in range(3): c=a@b
torch.cuda.synchronize();t=time.time()
for i in range(5): c=a@b
torch.cuda.synchronize();dt=(time.time()-t)/5
print('cuBLAS DGEMM 8192^3: %.2f TFLOP/s'%(2*8192**3/dt/1e12))
" >> gpurun_out/r6_gemm.log 2>&1
RSF_PROFILE=1 timeout 400 python tools/dev_scale.py 3 > gpurun_out/r6_scale3.log 2>&1; echo "exit $?" >> gpurun_out/r6_scale3.log
RSF_VERBOSE=2 RSF_PEEL_LEVELS=3 timeout 900 python tools/dev_scale.py 4 > gpurun_out/r6_scale4.log 2>&1; echo "exit $?" >> gpurun_out/r6_scale4.log
