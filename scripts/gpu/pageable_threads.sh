for t in 4 8 16; do echo "threads $t"; LSCAN_HOST_COPY_THREADS=$t LSCAN_HOST_CHUNK_MB=32 timeout 200 python scripts/pcie_lab.py pipe 2>&1 | tail -1; done
