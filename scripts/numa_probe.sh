#!/bin/bash
# GPU 0's NUMA node and the pinned-copy bandwidth with the process bound to
# each node's CPUs (pinned pages are first-touched on the binding node)
bus=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader -i 0 | tr 'A-Z' 'a-z' | sed 's/^0000//')
dev=$(ls -d /sys/bus/pci/devices/*${bus#0000} 2>/dev/null | head -1)
echo "gpu0 bus=$bus sysfs=$dev numa_node=$(cat $dev/numa_node 2>/dev/null) local_cpus=$(cat $dev/local_cpulist 2>/dev/null)"
nproc; ls -d /sys/devices/system/node/node* | wc -l
for n in /sys/devices/system/node/node*; do echo "$(basename $n): $(cat $n/cpulist)"; done
for n in /sys/devices/system/node/node*; do
  cpus=$(cat $n/cpulist)
  echo "== bound to $(basename $n) ($cpus)"
  taskset -c "$cpus" python scripts/pcie_bw.py
done
echo "== unbound"; python scripts/pcie_bw.py
