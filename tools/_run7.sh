T="python tools/stage_ab.py"
$T 1024 4 gpurun_out/a.npz
FV_PTAB=0 $T 1024 4 gpurun_out/b.npz
python tools/stage_ab.py --cmp gpurun_out/a.npz gpurun_out/b.npz
$T 4096 1 gpurun_out/c.npz 3
cd paper_1908_00041_b200 && cp libfavest_b200.so /tmp/main.so && cp libfavest_alt.so libfavest_b200.so && cd ..
echo "--- producers first"
$T 1024 4 gpurun_out/a2.npz
FV_PTAB=0 $T 1024 4 gpurun_out/b2.npz
$T 4096 1 gpurun_out/c2.npz 3
python tools/stage_ab.py --cmp gpurun_out/c.npz gpurun_out/c2.npz
cp /tmp/main.so paper_1908_00041_b200/libfavest_b200.so
rm -f gpurun_out/*.npz
