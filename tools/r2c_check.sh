# final-state check: GPU tests, smoke, bench (both arms), oracle-mode launch lists
mkdir -p gpurun_out
bash tools/r2_check.sh
python tools/oracle_prof.py 26 3 exp > gpurun_out/om_plain26.txt 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_oracle_launches_2p26.csv python tools/oracle_prof.py 26 1 exp > /dev/null 2>&1
python tools/oracle_prof.py 20 20 exp > gpurun_out/om_plain20.txt 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_oracle_launches_2p20.csv python tools/oracle_prof.py 20 1 exp > /dev/null 2>&1
