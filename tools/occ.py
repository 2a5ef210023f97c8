"""Report max active clusters for the GEMM kernels (cudaOccupancyMaxActiveClusters via ctypes to cudart)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
torch.cuda.init()
print(torch.cuda.get_device_properties(0))
