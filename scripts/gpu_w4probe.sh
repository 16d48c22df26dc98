mkdir -p gpurun_out
for v in "" _nocvt _nomma _cw16; do
  SUN_LIB=$PWD/paper_2603_02599_b200/libsun_b200$v.so timeout 300 python scripts/w4_probe.py > gpurun_out/w4probe$v.log 2>&1
done
for wg in 2 8; do SUN_W4_WGROUP=$wg timeout 300 python scripts/w4_probe.py > gpurun_out/w4probe_wg$wg.log 2>&1; done
SUN_W4_XSTAGES=4 timeout 300 python scripts/w4_probe.py > gpurun_out/w4probe_xs4.log 2>&1
tail -n 17 gpurun_out/w4probe*.log | grep -v "^{"
