bash tools/ab.sh ${1:-ab4} "PETRA_WGRAD_PRIO=0" "PETRA_WGRAD_PRIO=1" "PETRA_WGRAD_PRIO=2" "PETRA_WGRAD_PRIO=0" "PETRA_WGRAD_PRIO=1" "PETRA_WGRAD_PRIO=2"
python -c "import torch; print('priority range', torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream,'priority_range') else None)" 2>/dev/null
