"""B200-native plan-evaluation hot path of the Atlas/BubbleTea planner."""
