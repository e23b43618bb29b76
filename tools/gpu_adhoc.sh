cd $GRAFT_REPO_ROOT 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
rm -f gpurun_out/diag4.log
for c in C4z1.5 C4z1.0; do
echo "== $c" >> gpurun_out/diag4.log
CONFIG=$c PERLAUNCH=1 timeout 300 python tools/diag.py phj-gftr smj-gftr >> gpurun_out/diag4.log 2>&1
done
for c in C4z0.5 C2; do
echo "== $c" >> gpurun_out/diag4.log
CONFIG=$c timeout 300 python tools/diag.py phj-gftr smj-gftr >> gpurun_out/diag4.log 2>&1
done
grep -v " [012] wall" gpurun_out/diag4.log | grep "==\|scatter\| 3 wall"
