for mb in 1 2 3; do echo "MINB=$mb"; DICE_GATE_MINB=$mb python tools/mem_probe.py 2>&1 | head -1; done
