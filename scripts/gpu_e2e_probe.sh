# PCIe copy throughput and the per-p host-buffer overhead of the e2e path
cd $GRAFT_REPO_ROOT
O=gpurun_out/e2e
mkdir -p $O
timeout 300 python scripts/pcie_probe.py > $O/pcie.log 2>&1
timeout 600 python scripts/e2e_diag.py > $O/e2e_diag.log 2>&1
cat $O/pcie.log $O/e2e_diag.log
