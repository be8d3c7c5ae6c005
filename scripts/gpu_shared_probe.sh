# round 2: shared-table memory kinds (scripts/probes/shared_table_probe.cu)
R=gpurun_out/shared1; mkdir -p $R
P=build/probes/shared_table_probe
nvidia-smi -q | grep -i -A3 "addressing\|hmm" > $R/smi_addressing.txt 2>&1
cat /proc/driver/nvidia/version > $R/driver.txt 2>&1
cat /sys/module/nvidia_uvm/parameters/* > $R/uvm_params.txt 2>&1; ls /sys/module/nvidia_uvm/parameters/ >> $R/uvm_params.txt 2>&1
uname -a >> $R/driver.txt
for m in managed register hmm_anon hmm_memfd register_memfd hmm_anon_noadv hmm_memfd_noadv; do
  timeout 240 $P $m 16 >> $R/p16.jsonl 2>&1; echo "{\"mode_done\": \"$m\", \"rc\": $?}" >> $R/p16.jsonl
done
for m in managed hmm_memfd hmm_anon register_memfd; do
  timeout 400 $P $m 53 >> $R/p53.jsonl 2>&1; echo "{\"mode_done\": \"$m\", \"rc\": $?}" >> $R/p53.jsonl
done
