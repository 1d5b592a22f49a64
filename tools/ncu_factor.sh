# one ncu --set full capture of the factor kernel in the c3 bench geometry (after a plain run)
python tools/kt_probe.py ${KARGS:-3 full 0 3} > gpurun_out/plain_factor.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-factor_reg} -s ${SKIP:-2} -c ${COUNT:-1} \
    -o gpurun_out/${OUT:-prof_factor} python tools/kt_probe.py ${KARGS:-3 full 0 3} > gpurun_out/ncu_factor.log 2>&1
tail -3 gpurun_out/ncu_factor.log
