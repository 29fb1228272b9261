for rep in 1 2; do
EMS_P2_UNIT_MAJOR=0 EMS_P2_HSPLIT=1 python tools/energy.py --steps 150
EMS_P2_UNIT_MAJOR=1 EMS_P2_HSPLIT=2 python tools/energy.py --steps 150
done
