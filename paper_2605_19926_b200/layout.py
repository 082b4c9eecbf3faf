"""Engine ABI constants shared by the host layer and the CUDA library.

Values are part of the drop-in contract: they equal the reference's
``tilecast.backend.layout`` (/root/reference/pkg/src/tilecast/backend/layout.py:8-66)
and the ``TC_*`` macros in ``include/tilecast_b200.h``; ``_native`` asserts
the status / mode / capacity constants against the library's at import.
"""

# packed float constants, f64[FC_COUNT]  (layout.py:8-19)
FC_MOVE_SPEED, FC_RADIUS, FC_TURN_COS, FC_TURN_SIN, FC_ATTEN = 0, 1, 2, 3, 4
FC_GOAL_REWARD, FC_LIVING_REWARD, FC_HEALTH_DECAY, FC_HEALTH_RESTORE = 5, 6, 7, 8
FC_SPRITE_K, FC_MIN_SPRITE_DEPTH = 9, 10
FC_COUNT = 11

# packed int constants, i64[IC_COUNT]  (layout.py:22-25)
IC_MAX_STEPS, IC_GOAL_MODE, IC_USE_HEALTH = 0, 1, 2
IC_COUNT = 3

# action tags  (layout.py:28-35)
A_FORWARD, A_BACKWARD, A_TURN_LEFT, A_TURN_RIGHT = 0, 1, 2, 3
A_STRAFE_LEFT, A_STRAFE_RIGHT, A_NOOP = 4, 5, 6
A_COUNT = 7

# cell tags and entity kinds  (layout.py:38-45)
C_FLOOR, C_WALL, C_DOOR = 0, 1, 2
K_KEY, K_GOAL, K_MEDKIT = 0, 1, 2

# per-env kernel status  (layout.py:48-51, plus the device-side action check)
ST_OK, ST_ESCAPED, ST_STEP_BUDGET, ST_BAD_ACTION = 0, 1, 2, 3

# event bits, u32 per step  (layout.py:53-59)
EV_KEY_BASE_BIT, EV_DOOR_BASE_BIT = 0, 3
EV_MEDKIT_BIT, EV_GOAL_BIT, EV_DIED_BIT, EV_TRUNCATED_BIT = 6, 7, 8, 9

# batch kernel modes  (layout.py:61-62)
MODE_RESET, MODE_STEP = 0, 1

# fixed capacities  (layout.py:65-66)
MAX_ENTITIES = 64
MAX_DOORS = 32
