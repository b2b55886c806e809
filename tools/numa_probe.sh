nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
BUS=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-F' 'a-f' | sed 's/^0000//')
echo "bus $BUS" >> gpurun_out/topo.txt
for d in /sys/bus/pci/devices/*; do case "$d" in *${BUS#0000}*) echo "$d numa=$(cat $d/numa_node) cpus=$(cat $d/local_cpulist)" >> gpurun_out/topo.txt;; esac; done
lscpu | grep -i "numa\|socket\|model name" >> gpurun_out/topo.txt
nproc >> gpurun_out/topo.txt
python tools/pcie_duplex.py >> gpurun_out/topo.txt 2>&1
for n in 0 1; do echo "node $n" >> gpurun_out/topo.txt; numactl --cpunodebind=$n --membind=$n python tools/pcie_duplex.py >> gpurun_out/topo.txt 2>&1 || echo "no numactl" >> gpurun_out/topo.txt; done
