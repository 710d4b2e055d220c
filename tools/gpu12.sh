timeout 900 python -m pytest tests/test_gpu_tri.py tests/test_gpu_setup.py -q --tb=short -p no:cacheprovider > gpurun_out/pytest_r2v12.log 2>&1
timeout 600 compute-sanitizer --tool initcheck --print-limit 20 python tools/sanitize_driver.py > gpurun_out/sanitizer_initcheck2.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_initcheck2.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2404_14864_b200 as k
from paper_2404_14864_b200 import dist as D
for m, c in ((256, False), (512, True)):
    grid = k.CartesianGrid((-1.5,1.5,-1.5,1.5), m)
    rhs = torch.randn((m+1,m+1), dtype=torch.complex128 if c else torch.float64, device='cuda')
    for p in (1, 2, 4):
        D.solve_virtual(grid, 2j*m if c else 2.0*m, rhs, p, mode='carry')
print('carry ok')
" > gpurun_out/sanitizer_memcheck_carry.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer_memcheck_carry.log
