cd $GRAFT_REPO_ROOT
O=gpurun_out
for rep in 1 2; do
timeout 300 python tools/pcie_probe.py 2>/dev/null | sed "s|^|default |"
FXG_LIB=lib_alt/nosplit/libfxg.so timeout 300 python tools/pcie_probe.py 2>/dev/null | sed "s|^|nosplit |"
done > $O/r2x_pcie.log
cat $O/r2x_pcie.log
