for c in ppo_f32_I1B8T6E2M4 ppo_f32_I2B4T5E2M2 ppo_f64_I2B4T5E2M2 ppo_f64_I1B6T7E3M2; do
 echo "== $c default"; python tools/debug_case.py $c
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
