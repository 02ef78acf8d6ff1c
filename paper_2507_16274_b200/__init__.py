"""B200-native STWeaver planner + replay scorer (drop-in for the reference `memplan` API)."""
