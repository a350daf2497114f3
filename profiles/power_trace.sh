# SM clock and board power (nvidia-smi, 100 ms) while each config's scan runs back to back for ~1.5 s
for cfg in C5 C2 C3 C4; do
  nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 100 > /tmp/smi_$cfg.txt &
  SMI=$!
  SUSTAINED_SECONDS=1.5 python profiles/sustained_configs.py $cfg
  kill $SMI
  echo "  smi ($cfg): $(tr '\n' '|' < /tmp/smi_$cfg.txt)"
done
