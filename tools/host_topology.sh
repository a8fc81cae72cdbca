nvidia-smi topo -m 2>&1 | head -20
lscpu | grep -i "numa\|socket\|model name\|^CPU(s)"
cat /proc/self/status | grep -i cpus_allowed_list
ls /sys/devices/system/node/ | head
for n in /sys/devices/system/node/node*; do echo $n $(cat $n/cpulist) $(grep MemTotal $n/meminfo); done
cat /sys/bus/pci/devices/$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | tr 'A-Z' 'a-z' | sed 's/^0000//;s/^/0000/' | cut -c1-12)/numa_node 2>/dev/null
nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader
which numactl taskset || true
