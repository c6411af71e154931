for nw in 8 16; do echo "NW=$nw"; MD_FUSED_NW=$nw timeout 500 python scripts/c4_breakdown.py | tail -4; done
