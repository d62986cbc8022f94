BT_BASIS_DEBUG=1 timeout 600 python tools/prof_c3.py > gpurun_out/prof_c3c.log 2>&1; grep -n "cholqr\|subspace\|mode_basis\|total\|eigh\|unfold" gpurun_out/prof_c3c.log | head -40
BT_BASIS_DEBUG=1 timeout 600 python tools/prof_c2.py > gpurun_out/prof_c2d.log 2>&1; grep -n "subspace\|mode_basis\|total\|eigh\|complete" gpurun_out/prof_c2d.log | head -30
