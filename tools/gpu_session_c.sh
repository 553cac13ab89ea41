# organisations of the depth solve on cfg3 (CFL_IMEX 2 and MCFL-only) and on one 2^22-cell member
for m in 0 1 3 4; do echo "== cfg3 mode $m"; timeout 120 python tools/cl_probe.py 4096 20 $m; done
for m in 1 3 4; do echo "== cfg3 MCFL-only mode $m"; timeout 120 python tools/cl_probe.py 4096 20 $m 4096 0; done
for m in 0 3; do echo "== 1 x 2^22 mode $m"; timeout 120 python tools/cl_probe.py 1 20 $m 4194304; done
echo "== 1 x 2^22 MCFL-only spike"; timeout 120 python tools/cl_probe.py 1 20 3 4194304 0
