# multicast (NVLS) support probe on the one-GPU box
timeout -s KILL 120 python tools/probe_multicast.py 2>&1 | tail -8
nvidia-smi topo -m 2>&1 | head -5
