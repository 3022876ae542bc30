# A/B of the gang truncation variants (HCOV_GANG_QR=0 Householder, 1 CholeskyQR3) at 524K
export HCOV_WATCHDOG_S=600
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/ab.log
for gm in 0 1; do
  HCOV_GANG_QR=$gm timeout 900 python tools/timeline.py run tl_gm$gm 524288 0.5 0.1 1e-6 20 > gpurun_out/ab_gm$gm.log 2>&1
  echo "gm$gm rc=$?" >> gpurun_out/ab.log
done
