"""Slab-emulation probe: planck face unsplit vs split into G row slabs (all ranks on this GPU)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import bench
for G in (2, 4, 8):
    print(json.dumps(bench._slab_probe(torch.device("cuda:0"), G=G)), flush=True)
