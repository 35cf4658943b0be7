python tools/oracle_prof.py 26 2 exp > gpurun_out/om_plain.txt 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:words_cls -c 1 -o gpurun_out/r02_words_cls python tools/oracle_prof.py 26 2 exp > gpurun_out/om_ncu.log 2>&1
